// librl host code: error state, launch counters, optional event timing, device checks.
// Included once, in order, by rl_api.cu (a single translation unit); everything
// here has internal linkage.
#pragma once

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

// ---------------------------------------------------- optional event timing
struct ProfRec {
  int kernel;
  cudaEvent_t a, b;
};
thread_local bool g_prof = false;
thread_local std::vector<ProfRec> g_prof_recs;
thread_local std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launch with events when timing is enabled.
struct ProfScope {
  int kernel;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int k, cudaStream_t s) : kernel(k), st(s) {
    if (g_prof) {
      a = prof_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      g_prof_recs.push_back({kernel, a, b});
    }
  }
};

rl_status fail(rl_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

#define RL_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(RL_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define RL_CHECK_LAUNCH()                                                                      \
  do {                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ != cudaSuccess) return fail(RL_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e_)); \
    ++g_launches;                                                                              \
  } while (0)

#define RL_TRY(x)                  \
  do {                             \
    rl_status s_ = (x);            \
    if (s_ != RL_OK) return s_;    \
  } while (0)

#define RL_NONNULL(p) \
  if (!(p)) return fail(RL_ERR_INVALID_ARGUMENT, "%s is NULL", #p)

// ------------------------------------------------------------- device info
struct DevInfo {
  int sms = 0;
  bool ok = false;
};

rl_status device_info(DevInfo& d) {
  int dev = 0;
  RL_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static DevInfo cache[64];
  static bool have[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return fail(RL_ERR_UNSUPPORTED, "device index %d out of range", dev);
  if (!have[dev]) {
    int major = 0, minor = 0, sms = 0;
    RL_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    RL_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    RL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev].sms = sms;
    cache[dev].ok = (major == 10 && minor == 0);
    have[dev] = true;
  }
  d = cache[dev];
  if (!d.ok) return fail(RL_ERR_UNSUPPORTED, "librl is built for sm_100a (B200); device %d is not compute 10.0", dev);
  return RL_OK;
}

}  // namespace
