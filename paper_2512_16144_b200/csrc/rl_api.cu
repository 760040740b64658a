// librl host side: argument validation, workspace carving, TMA tensor maps and
// kernel launches behind the C ABI of include/rl.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "../../include/rl.h"
#include "rl_gemm.cuh"
#include "rl_small.cuh"

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

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

rl_status get_encode(EncodeTiledFn& fn) {
  static EncodeTiledFn cached = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) cached = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!cached) return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(err));
  fn = cached;
  return RL_OK;
}

// 2-D row-major tensor [outer][inner], 128-byte swizzle, zero fill out of bounds.
rl_status make_map(CUtensorMap* m, const void* ptr, bool f32, int64_t inner, int64_t outer, int64_t row_elems,
                   int box_inner, int box_outer) {
  EncodeTiledFn enc;
  rl_status s = get_encode(enc);
  if (s != RL_OK) return s;
  const int esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer > 0 ? outer : 1)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_elems * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for [%lld x %lld] box %dx%d", (int)r,
                (long long)outer, (long long)inner, box_outer, box_inner);
  return RL_OK;
}

// ----------------------------------------------------------------- GEMMs
// CTA-pair (cta_group::2, 256x256 tiles) by default; RL_CTA_GROUP=1 selects the
// single-CTA 128x256 variant (kept for A/B measurements and as a fallback).
int cta_group() {
  static int cg = [] {
    const char* e = getenv("RL_CTA_GROUP");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return cg;
}

// Raster group (in m-blocks) per GEMM: tiles walk n inside groups of this many
// m-blocks. Defaults chosen from the sweep in DESIGN.md §5; RL_GROUP_M_<K>
// overrides (K in FWD, DZ, DH, DW) for measurements.
int group_m_for(int kid, int dflt) {
  static int cache[16];
  static bool init[16] = {};
  if (!init[kid]) {
    const char* names[16] = {nullptr, "RL_GROUP_M_FWD", nullptr, nullptr, nullptr, "RL_GROUP_M_DZ",
                             "RL_GROUP_M_DH", "RL_GROUP_M_DW"};
    const char* e = names[kid] ? getenv(names[kid]) : nullptr;
    cache[kid] = (e && atoi(e) > 0) ? atoi(e) : dflt;
    init[kid] = true;
  }
  return cache[kid];
}

// Soft k-barrier between producers (see EpiParams::sync_*): every RL_SYNC_EVERY
// k-blocks (default 32; 0 = off), at most RL_SYNC_SLACK sync points of lead
// (default 2). Keeping the CTAs that share operands inside one L2 window cuts
// K5/K6 DRAM reads by ~1/3 and lets the power-capped clock rise (~6% per step,
// profiles/r01/). Correctness never depends on it (the wait is bounded).
// Per-GEMM overrides: RL_SYNC_EVERY_<K>, RL_SYNC_SLACK_<K> (K in FWD, DZ, DH, DW, NS).
const char* kid_suffix(int kid) {
  switch (kid) {
    case RL_K_FWD_GEMM: return "FWD";
    case RL_K_DZ_GEMM: return "DZ";
    case RL_K_DH_GEMM: return "DH";
    case RL_K_DW_GEMM: return "DW";
    case RL_K_NS_GEMM: return "NS";
    default: return "OTHER";
  }
}
int env_int(const char* base, int kid, int dflt) {
  char name[64];
  snprintf(name, sizeof(name), "%s_%s", base, kid_suffix(kid));
  const char* e = getenv(name);
  if (!e) e = getenv(base);
  return e ? atoi(e) : dflt;
}
int sync_every_for(int kid) {
  static int cache[32];
  static bool init[32] = {};
  if (kid < 0 || kid >= 32) return 0;
  if (!init[kid]) {
    cache[kid] = env_int("RL_SYNC_EVERY", kid, 32);
    init[kid] = true;
  }
  return cache[kid];
}
// Wide 256 x 512 pair tiles (NB = 2, rl_gemm.cuh): RL_WIDE[_<K>] = 0/1, default on
// for K1 (FWD), K5 (DH), K6 (DW) and the Newton-Schulz GEMMs (NS: 41.0 -> 38.6 ms); RL_SKEW = 0/2/3 k-blocks of block-0-first MMA
// order at both ends of a tile (default 3), which hides the epilogue of one TMEM
// half. K4 (DZ) stays narrow: its exp + bf16-store epilogue per half is longer
// than that cover (measured: K4 15.6 -> 17.9 ms wide, K1 15.6 -> 15.2 ms).
bool wide_for(int kid) {
  static int cache[32];
  static bool init[32] = {};
  if (kid < 0 || kid >= 32) return false;
  if (!init[kid]) {
    const bool dflt = kid == RL_K_FWD_GEMM || kid == RL_K_DH_GEMM || kid == RL_K_DW_GEMM || kid == RL_K_NS_GEMM;
    cache[kid] = env_int("RL_WIDE", kid, dflt ? 1 : 0);
    init[kid] = true;
  }
  return cache[kid] != 0;
}
int skew() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RL_SKEW");
    v = e ? atoi(e) : 3;
    if (v != 0 && v != 2) v = 3;
  }
  return v;
}
int sync_slack_for(int kid) {
  static int cache[32];
  static bool init[32] = {};
  if (kid < 0 || kid >= 32) return 2;
  if (!init[kid]) {
    cache[kid] = env_int("RL_SYNC_SLACK", kid, 2);
    init[kid] = true;
  }
  return cache[kid];
}
constexpr int kMaxSyncPoints = 1 << 16;
thread_local uint32_t* g_sync_ctr = nullptr;  // set per call from the workspace

template <int CG, int NB>
constexpr int stages_for() {
  return CG == 2 ? (NB == 2 ? 4 : 6) : 4;
}

template <int MODE, bool A_MN, bool B_MN, int CG, int NB = 1, int SKEW = 0>
rl_status launch_gemm_cg(int kid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t M,
                         int64_t N, int64_t K, int group_m, const rl::EpiParams& ep, int sms, cudaStream_t st,
                         int k_splits = 1, int split_rows = 0, const int* dyn_count = nullptr, int dyn_mode = 0) {
  constexpr int S = stages_for<CG, NB>();
  auto kern = rl::gemm_kernel<MODE, A_MN, B_MN, CG, S, NB, SKEW>;
  constexpr int smem = rl::gemm_smem_bytes<CG, S, false, NB>();
  static_assert(smem <= 232448, "dynamic shared memory over 227 KB");
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    RL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  using TL = rl::Tiling<CG>;
  rl::GemmShape sh;
  sh.m_blocks = static_cast<int>((M + TL::TILE_M - 1) / TL::TILE_M);
  sh.n_blocks = static_cast<int>((N + rl::BN * NB - 1) / (rl::BN * NB));
  sh.k_blocks = static_cast<int>((K + rl::BK - 1) / rl::BK);
  sh.group_m = group_m;
  if (sh.k_blocks == 0) return fail(RL_ERR_SHAPE, "GEMM with K = 0");
  if (k_splits < 1) k_splits = 1;
  if (k_splits > sh.k_blocks) k_splits = sh.k_blocks;
  sh.k_per_split = (sh.k_blocks + k_splits - 1) / k_splits;
  sh.k_splits = (sh.k_blocks + sh.k_per_split - 1) / sh.k_per_split;
  sh.split_rows = split_rows;
  sh.dyn_count = dyn_count;
  sh.dyn_mode = dyn_count ? dyn_mode : 0;
  if (sh.k_splits > 1 && (MODE == rl::EPI_LSE || MODE == rl::EPI_DZ || MODE == rl::EPI_F32_NVLS))
    return fail(RL_ERR_UNSUPPORTED, "split-K needs a plain store epilogue");
  const int64_t tiles = static_cast<int64_t>(sh.m_blocks) * sh.n_blocks * sh.k_splits;
  const int units = static_cast<int>(tiles < sms / CG ? tiles : sms / CG);
  rl::EpiParams ep2 = ep;
  ep2.sync_every = 0;
  if (g_sync_ctr && sync_every_for(kid) > 0) {
    const int64_t max_tiles = (tiles + units - 1) / units;
    const int se = sync_every_for(kid);
    const int64_t max_sync = (max_tiles * sh.k_blocks - 1) / se;
    if (max_sync > 0 && max_sync < kMaxSyncPoints) {
      RL_CUDA(cudaMemsetAsync(g_sync_ctr, 0, static_cast<size_t>(max_sync + 1) * 4, st));
      ep2.sync_ctr = g_sync_ctr;
      ep2.sync_every = se;
      ep2.sync_slack = sync_slack_for(kid);
      ep2.max_sync = static_cast<int>(max_sync);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(rl::GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  {
    ProfScope ps(kid, st);
    RL_CUDA(cudaLaunchKernelEx(&cfg, kern, a, b, c, sh, ep2));
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

template <int MODE, bool A_MN, bool B_MN>
rl_status launch_gemm(int kid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t M, int64_t N,
                      int64_t K, int group_m, const rl::EpiParams& ep, int sms, cudaStream_t st, int k_splits = 1,
                      int split_rows = 0, const int* dyn_count = nullptr, int dyn_mode = 0) {
  if (M <= 0 || N <= 0) return RL_OK;
  // wide tiles only where a tile covers at least two 256-column blocks
  if (cta_group() == 2 && wide_for(kid) && N > rl::BN) {
    switch (skew()) {
      case 0:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 0>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                         split_rows, dyn_count, dyn_mode);
      case 2:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 2>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                         split_rows, dyn_count, dyn_mode);
      default:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 3>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                         split_rows, dyn_count, dyn_mode);
    }
  }
  if (cta_group() == 2)
    return launch_gemm_cg<MODE, A_MN, B_MN, 2>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
                                               dyn_count, dyn_mode);
  return launch_gemm_cg<MODE, A_MN, B_MN, 1>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
                                             dyn_count, dyn_mode);
}

// Grouped GEMM (MoE experts): the tile count is only known on the device (it
// depends on the group offsets), so the grid is sized from an upper bound.
template <int CG>
rl_status launch_grouped_cg(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t rows,
                            int64_t N, int64_t K, int n_groups, const rl::EpiParams& ep, int sms, cudaStream_t st) {
  constexpr int S = CG == 2 ? 5 : 3;
  auto kern = rl::gemm_kernel<rl::EPI_BF16_GROUPED, false, false, CG, S>;
  constexpr int smem = rl::gemm_smem_bytes<CG, S, true>();
  static bool attr_set = false;
  if (!attr_set) {
    RL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  using TL = rl::Tiling<CG>;
  rl::GemmShape sh = {};
  sh.n_blocks = static_cast<int>((N + rl::BN - 1) / rl::BN);
  sh.m_blocks = static_cast<int>((rows + TL::TILE_M - 1) / TL::TILE_M) + n_groups;  // bound on group m-blocks
  sh.k_blocks = static_cast<int>((K + rl::BK - 1) / rl::BK);
  sh.group_m = 1;
  sh.k_splits = 1;
  sh.k_per_split = sh.k_blocks;
  const int64_t tiles = static_cast<int64_t>(sh.m_blocks) * sh.n_blocks;
  const int units = static_cast<int>(tiles < sms / CG ? tiles : sms / CG);
  rl::EpiParams e = ep;
  e.sync_every = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(rl::GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  {
    ProfScope ps(RL_K_GROUPED_GEMM, st);
    RL_CUDA(cudaLaunchKernelEx(&cfg, kern, a, b, c, sh, e));
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

// Rows of A staged per CTA per tile (the TMA box height for A loads).
constexpr int kARows = 128;

// ------------------------------------------------------------ workspace
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Carve {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = align_up(off, 1024);
    off = o + bytes;
    return o;
  }
};

struct WsLayout {
  size_t partials, lse, coef, rp, sync, dz, end;
  // sparse backward (rows with coef != 0): compact index, per-row vectors, counts,
  // gathered hidden rows and one chunk of compact dH
  size_t idx, coef_c, lse_c, tgt_c, invt_c, blk_counts, chunk_counts, h_c, dh_c;
  int64_t n_tiles_v, ldz, chunk;
};

int64_t n_vocab_tiles(const rl_lm_shape* s) { return (s->V_local + rl::BN - 1) / rl::BN; }

WsLayout ws_layout(const rl_lm_shape* s, int32_t R, int64_t chunk_rows) {
  WsLayout w;
  Carve c;
  const int64_t T = s->T > 0 ? s->T : 0;
  w.n_tiles_v = n_vocab_tiles(s);
  w.ldz = (s->V_local + 7) / 8 * 8;
  w.chunk = (chunk_rows <= 0 || chunk_rows > T) ? T : chunk_rows;
  w.partials = c.take(static_cast<size_t>(w.n_tiles_v) * T * 16);
  w.lse = c.take(static_cast<size_t>(T) * 4);
  w.coef = c.take(static_cast<size_t>(T) * 4);
  w.rp = c.take(static_cast<size_t>(R > 0 ? R : 1) * sizeof(rl::RolloutPartial));
  w.sync = c.take(static_cast<size_t>(kMaxSyncPoints) * 4);
  w.dz = c.take(static_cast<size_t>(w.chunk) * w.ldz * 2);
  const int64_t Tp = (T + 255) / 256 * 256 + 256;  // compact rows + zero padding (gather_rows_kernel)
  w.idx = c.take(static_cast<size_t>(Tp) * 4);
  w.coef_c = c.take(static_cast<size_t>(Tp) * 4);
  w.lse_c = c.take(static_cast<size_t>(Tp) * 4);
  w.tgt_c = c.take(static_cast<size_t>(Tp) * 4);
  w.invt_c = c.take(static_cast<size_t>(Tp) * 4);
  w.blk_counts = c.take(static_cast<size_t>((T + rl::COMPACT_ROWS - 1) / rl::COMPACT_ROWS + 1) * 4);
  w.chunk_counts = c.take(static_cast<size_t>((T + (w.chunk > 0 ? w.chunk : 1) - 1) / (w.chunk > 0 ? w.chunk : 1) + 2) * 4);
  w.h_c = c.take(static_cast<size_t>(Tp) * s->H * 2);
  w.dh_c = c.take(static_cast<size_t>((w.chunk + 255) / 256 * 256) * s->H * 4);
  w.end = align_up(c.off, 1024);
  return w;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

rl_status check_shape(const rl_lm_shape* s) {
  if (!s) return fail(RL_ERR_INVALID_ARGUMENT, "shape is NULL");
  if (s->T < 0 || s->T > (int64_t(1) << 31) - 1) return fail(RL_ERR_SHAPE, "T = %lld out of range", (long long)s->T);
  if (s->H <= 0 || s->H % 8 != 0 || s->H > 65536) return fail(RL_ERR_SHAPE, "H = %lld must be a positive multiple of 8 <= 65536", (long long)s->H);
  if (s->V_local <= 0 || s->V_local > (int64_t(1) << 31) - 1) return fail(RL_ERR_SHAPE, "V_local = %lld out of range", (long long)s->V_local);
  if (s->vocab_offset < 0 || s->V_global < s->vocab_offset + s->V_local)
    return fail(RL_ERR_SHAPE, "vocab_offset %lld + V_local %lld exceeds V_global %lld", (long long)s->vocab_offset,
                (long long)s->V_local, (long long)s->V_global);
  if (!(s->inv_temperature > 0.f) || !isfinite(s->inv_temperature))
    return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be finite and > 0");
  if (s->inv_temperature_rows && (reinterpret_cast<uintptr_t>(s->inv_temperature_rows) & 3u))
    return fail(RL_ERR_ALIGNMENT, "inv_temperature_rows must be 4-byte aligned");
  return RL_OK;
}

static_assert(sizeof(rl_lm_shape) == 56, "rl_lm_shape layout (binding mirrors it)");
static_assert(sizeof(rl_loss_params) == 40, "rl_loss_params layout (binding mirrors it)");
static_assert(sizeof(rl_loss_report) == 48, "rl_loss_report layout (binding mirrors it)");

rl_status check_params(const rl_loss_params* p) {
  if (!p) return fail(RL_ERR_INVALID_ARGUMENT, "params is NULL");
  if (!(p->alpha > 0.f) || !(p->alpha <= 1.f) || !(p->beta >= 1.f) || !isfinite(p->beta))
    return fail(RL_ERR_INVALID_ARGUMENT, "need 0 < alpha <= 1 <= beta (got alpha=%g beta=%g)", p->alpha, p->beta);
  if (!(p->guard_threshold >= 0.f) || !isfinite(p->guard_threshold))
    return fail(RL_ERR_INVALID_ARGUMENT, "guard_threshold must be finite and >= 0");
  if (!(p->loss_denominator > 0.0) || !isfinite(p->loss_denominator))
    return fail(RL_ERR_INVALID_ARGUMENT, "loss_denominator must be finite and > 0");
  if (p->num_rollouts < 1) return fail(RL_ERR_INVALID_ARGUMENT, "num_rollouts must be >= 1");
  if (p->variant < RL_LOSS_ICEPOP || p->variant > RL_LOSS_GSPO)
    return fail(RL_ERR_INVALID_ARGUMENT, "unknown loss variant %d", p->variant);
  if (!isfinite(p->kl_tau)) return fail(RL_ERR_INVALID_ARGUMENT, "kl_tau must be finite");
  if (p->kl_set < RL_KL_MASKED || p->kl_set > RL_KL_ALL)
    return fail(RL_ERR_INVALID_ARGUMENT, "unknown kl_set %d", p->kl_set);
  return RL_OK;
}

#define RL_TRY(x)                  \
  do {                             \
    rl_status s_ = (x);            \
    if (s_ != RL_OK) return s_;    \
  } while (0)

#define RL_NONNULL(p) \
  if (!(p)) return fail(RL_ERR_INVALID_ARGUMENT, "%s is NULL", #p)

// K1 (+ K2): forward over the local shard. If `merged` is non-null, write one
// merged partial per row; else write logprob/entropy/lse.
rl_status forward_impl(const rl_lm_shape* s, const uint16_t* hidden, const uint16_t* w, const int32_t* targets,
                       float* logprob, float* entropy, float* lse, float4* merged, uint8_t* ws, const WsLayout& L,
                       int sms, cudaStream_t st) {
  const int64_t T = s->T;
  if (T == 0) return RL_OK;
  CUtensorMap ta, tb;
  RL_TRY(make_map(&ta, hidden, false, s->H, T, s->H, 64, kARows));
  RL_TRY(make_map(&tb, w, false, s->H, s->V_local, s->H, 64, rl::BN / cta_group()));
  rl::EpiParams ep = {};
  ep.rows = T;
  ep.cols = s->V_local;
  ep.inv_temperature = s->inv_temperature;
  ep.scale_log2 = s->inv_temperature * 1.4426950408889634f;
  ep.invt_rows = s->inv_temperature_rows;
  ep.targets = targets;
  ep.vocab_offset = s->vocab_offset;
  float4* parts = reinterpret_cast<float4*>(ws + L.partials);
  ep.partials = parts;
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + L.sync);
  RL_TRY((launch_gemm<rl::EPI_LSE, false, false>(RL_K_FWD_GEMM, ta, tb, ta, T, s->V_local, s->H, group_m_for(RL_K_FWD_GEMM, 16), ep, sms, st)));
  const int blocks = static_cast<int>((T + rl::MERGE_ROWS - 1) / rl::MERGE_ROWS);
  {
    ProfScope ps(RL_K_MERGE, st);
    rl::merge_partials_kernel<<<blocks, 256, 0, st>>>(parts, static_cast<int>(L.n_tiles_v), T, logprob, entropy,
                                                        lse, merged);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status loss_impl(const rl_loss_params* p, int64_t T, int64_t V_global, const float* logprob, const float* infer,
                    const int32_t* targets, const float* adv, const int32_t* offsets, const uint8_t* loss_mask,
                    float* coef, uint8_t* keep, uint8_t* guarded, rl_loss_report* rep, rl::RolloutPartial* rp,
                    cudaStream_t st) {
  rl::LossArgs a;
  a.variant = p->variant;
  a.kl_set = p->kl_set;
  a.kl_w = static_cast<double>(p->kl_tau) / p->loss_denominator;
  a.alpha = p->alpha;
  a.beta = p->beta;
  a.guard = p->guard_threshold;
  a.inv_D = 1.0 / p->loss_denominator;
  a.R = p->num_rollouts;
  a.T = T;
  a.V_global = V_global;
  a.logprob = logprob;
  a.infer = infer;
  a.targets = targets;
  a.adv = adv;
  a.offsets = offsets;
  a.loss_mask = loss_mask;
  a.coef = coef;
  a.keep = keep;
  a.guarded = guarded;
  a.rp = rp;
  {
    ProfScope ps(RL_K_LOSS, st);
    rl::loss_coef_kernel<<<p->num_rollouts, 256, 0, st>>>(a);
  }
  RL_CHECK_LAUNCH();
  {
    ProfScope ps(RL_K_FINALIZE, st);
    rl::loss_finalize_kernel<<<1, 32, 0, st>>>(rp, p->num_rollouts, rep);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

// K4 -> K5 -> K6 per chunk of rows.
// Fill the NVLS fields of an epilogue from the caller's descriptor; the
// multicast VA is offset like the local output pointer `local`.
void set_nvls(rl::EpiParams& e, const rl_nvls_reduce* n, const float* local) {
  (void)local;
  e.nvls_mc = static_cast<float*>(n->multicast);
  for (int r = 0; r < rl::NVLS_MAX_RANKS; ++r) e.nvls_flags[r] = n->flags[r];
  e.nvls_rank = n->rank;
  e.nvls_world = n->world;
  e.nvls_epoch = n->epoch;
  e.nvls_lag = n->lag > 0 ? n->lag : 2;
}

rl_status check_nvls(const rl_nvls_reduce* n, const char* what) {
  if (!n) return RL_OK;
  if (!n->multicast) return fail(RL_ERR_INVALID_ARGUMENT, "%s: multicast VA is NULL", what);
  if (n->world < 2 || n->world > RL_NVLS_MAX_RANKS || n->rank < 0 || n->rank >= n->world)
    return fail(RL_ERR_INVALID_ARGUMENT, "%s: need 2 <= world <= %d and 0 <= rank < world", what, RL_NVLS_MAX_RANKS);
  for (int r = 0; r < n->world; ++r)
    if (!n->flags[r]) return fail(RL_ERR_INVALID_ARGUMENT, "%s: flags[%d] is NULL", what, r);
  if (n->epoch == 0) return fail(RL_ERR_INVALID_ARGUMENT, "%s: epoch must be > 0 (flags start at 0)", what);
  return RL_OK;
}

// Sparse backward: the same K4 -> K6 -> K5 over the rows whose coefficient is
// non-zero only (their order kept). Row counts live on the device: the GEMMs read
// them at start (dyn_mode), so nothing synchronises the host.
rl_status bwd_sparse_impl(const rl_lm_shape* s, const uint16_t* hidden, const uint16_t* w, const int32_t* targets,
                          const float* lse, const float* coef, uint16_t* dh, float* dh32, float* dw,
                          int accumulate_dw, uint8_t* ws, const WsLayout& L, int sms, cudaStream_t st, int phases,
                          const rl_nvls_reduce* dw_nvls) {
  const int64_t T = s->T, H = s->H, V = s->V_local;
  const int64_t chunk = L.chunk;
  const int n_chunks = static_cast<int>((T + chunk - 1) / chunk);
  uint16_t* dz = reinterpret_cast<uint16_t*>(ws + L.dz);
  int32_t* idx = reinterpret_cast<int32_t*>(ws + L.idx);
  float* coef_c = reinterpret_cast<float*>(ws + L.coef_c);
  float* lse_c = reinterpret_cast<float*>(ws + L.lse_c);
  int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + L.tgt_c);
  float* invt_c = reinterpret_cast<float*>(ws + L.invt_c);
  int* blk = reinterpret_cast<int*>(ws + L.blk_counts);
  int* cc = reinterpret_cast<int*>(ws + L.chunk_counts);  // [n_chunks] per chunk, [n_chunks] total
  uint16_t* h_c = reinterpret_cast<uint16_t*>(ws + L.h_c);
  uint8_t* dh_c = ws + L.dh_c;
  if (phases & RL_BWD_DU) {
    const int nb = static_cast<int>((T + rl::COMPACT_ROWS - 1) / rl::COMPACT_ROWS);
    {
      ProfScope ps(RL_K_COMPACT, st);
      rl::compact_count_kernel<<<nb, 256, 0, st>>>(coef, T, blk);
    }
    RL_CHECK_LAUNCH();
    {
      ProfScope ps(RL_K_COMPACT, st);
      rl::compact_write_kernel<<<nb, 256, 0, st>>>(coef, lse, targets, T, blk, nb, chunk, idx, coef_c, lse_c, tgt_c,
                                                   cc, n_chunks, s->inv_temperature_rows, invt_c);
    }
    RL_CHECK_LAUNCH();
    {
      ProfScope ps(RL_K_COMPACT, st);
      rl::gather_rows_kernel<<<8 * sms, 256, 0, st>>>(hidden, H, idx, cc + n_chunks, 256, (T + 255) / 256 * 256 + 256,
                                                      h_c, coef_c, lse_c, tgt_c,
                                                      s->inv_temperature_rows ? invt_c : nullptr);
    }
    RL_CHECK_LAUNCH();
  }
  CUtensorMap t_w_k, t_w_mn, t_dw;
  RL_TRY(make_map(&t_w_k, w, false, H, V, H, 64, rl::BN / cta_group()));
  RL_TRY(make_map(&t_w_mn, w, false, H, V, H, 64, 64));
  if (dw) RL_TRY(make_map(&t_dw, dw, true, H, V, H, 32, 32));
  if ((phases & RL_BWD_DH) && (dh || dh32))
    RL_CUDA(cudaMemsetAsync(dh ? static_cast<void*>(dh) : static_cast<void*>(dh32), 0,
                            static_cast<size_t>(T) * H * (dh ? 2 : 4), st));
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int64_t c0 = ch * chunk;
    const int64_t rows = (T - c0 < chunk) ? (T - c0) : chunk;   // upper bound on this chunk's compact rows
    const int* cnt = cc + ch;
    const uint16_t* hc = h_c + c0 * H;
    CUtensorMap t_h_k, t_dz_st, t_dz_k, t_dz_mn, t_h_mn, t_dh;
    if (phases & RL_BWD_DU) {
      RL_TRY(make_map(&t_h_k, hc, false, H, rows, H, 64, kARows));
      RL_TRY(make_map(&t_dz_st, dz, false, V, rows, L.ldz, 64, 32));
      rl::EpiParams ep = {};
      ep.rows = rows;
      ep.cols = V;
      ep.inv_temperature = s->inv_temperature;
      ep.scale_log2 = s->inv_temperature * 1.4426950408889634f;
      ep.targets = tgt_c + c0;
      ep.vocab_offset = s->vocab_offset;
      ep.lse = lse_c + c0;
      ep.coef = coef_c + c0;
      ep.invt_rows = s->inv_temperature_rows ? invt_c + c0 : nullptr;
      RL_TRY((launch_gemm<rl::EPI_DZ, false, false>(RL_K_DZ_GEMM, t_h_k, t_w_k, t_dz_st, rows, V, H,
                                                    group_m_for(RL_K_DZ_GEMM, 16), ep, sms, st, 1, 0, cnt, 1)));
    }
    if ((phases & RL_BWD_DW) && dw) {
      RL_TRY(make_map(&t_dz_mn, dz, false, V, rows, L.ldz, 64, 64));
      RL_TRY(make_map(&t_h_mn, hc, false, H, rows, H, 64, 64));
      rl::EpiParams e6 = {};
      e6.rows = V;
      e6.cols = H;
      if (dw_nvls) {
        set_nvls(e6, dw_nvls, dw);
        RL_TRY((launch_gemm<rl::EPI_F32_NVLS, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                            group_m_for(RL_K_DW_GEMM, 8), e6, sms, st, 1, 0, cnt, 2)));
      } else if (ch == 0 && !accumulate_dw) {
        RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                     group_m_for(RL_K_DW_GEMM, 8), e6, sms, st, 1, 0, cnt, 2)));
      } else {
        RL_TRY((launch_gemm<rl::EPI_F32_ADD, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                         group_m_for(RL_K_DW_GEMM, 8), e6, sms, st, 1, 0, cnt, 2)));
      }
    }
    if ((phases & RL_BWD_DH) && (dh || dh32)) {
      RL_TRY(make_map(&t_dz_k, dz, false, V, rows, L.ldz, 64, kARows));
      rl::EpiParams e5 = {};
      e5.rows = rows;
      e5.cols = H;
      if (dh) {
        RL_TRY(make_map(&t_dh, dh_c, false, H, rows, H, 64, 32));
        RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                       group_m_for(RL_K_DH_GEMM, 8), e5, sms, st, 1, 0, cnt, 1)));
      } else {
        RL_TRY(make_map(&t_dh, dh_c, true, H, rows, H, 32, 32));
        RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                      group_m_for(RL_K_DH_GEMM, 8), e5, sms, st, 1, 0, cnt, 1)));
      }
      {
        ProfScope ps(RL_K_COMPACT, st);
        rl::scatter_rows_kernel<<<8 * sms, 256, 0, st>>>(dh_c, H * (dh ? 2 : 4), idx + c0, cnt,
                                                         dh ? reinterpret_cast<uint8_t*>(dh)
                                                            : reinterpret_cast<uint8_t*>(dh32));
      }
      RL_CHECK_LAUNCH();
    }
  }
  return RL_OK;
}

// K4 -> K6 -> K5 per chunk of rows (dW first, so a caller can overlap its
// reduction with dH). `phases` selects which run (RL_BWD_* bits).
rl_status bwd_impl(const rl_lm_shape* s, const uint16_t* hidden, const uint16_t* w, const int32_t* targets,
                   const float* lse, const float* coef, uint16_t* dh, float* dh32, float* dw, int accumulate_dw,
                   uint8_t* ws, const WsLayout& L, int sms, cudaStream_t st, int phases = RL_BWD_ALL,
                   const rl_nvls_reduce* dw_nvls = nullptr, const rl_nvls_reduce* dh_nvls = nullptr) {
  const int64_t T = s->T, H = s->H, V = s->V_local;
  if (T == 0) {
    if (dw && !accumulate_dw) RL_CUDA(cudaMemsetAsync(dw, 0, static_cast<size_t>(V) * H * 4, st));
    return RL_OK;
  }
  uint16_t* dz = reinterpret_cast<uint16_t*>(ws + L.dz);
  const int64_t chunk = L.chunk;
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + L.sync);
  if (!(phases & RL_BWD_DENSE) && !dh_nvls)
    return bwd_sparse_impl(s, hidden, w, targets, lse, coef, dh, dh32, dw, accumulate_dw, ws, L, sms, st, phases,
                           dw_nvls);
  CUtensorMap t_h_k, t_w_k, t_dz_st, t_dz_k, t_w_mn, t_dh, t_dz_mn, t_h_mn, t_dw;
  RL_TRY(make_map(&t_w_k, w, false, H, V, H, 64, rl::BN / cta_group()));
  RL_TRY(make_map(&t_w_mn, w, false, H, V, H, 64, 64));
  if (dw) RL_TRY(make_map(&t_dw, dw, true, H, V, H, 32, 32));
  for (int64_t c0 = 0; c0 < T; c0 += chunk) {
    const int64_t rows = (T - c0 < chunk) ? (T - c0) : chunk;
    const uint16_t* hc = hidden + c0 * H;
    RL_TRY(make_map(&t_h_k, hc, false, H, rows, H, 64, kARows));
    RL_TRY(make_map(&t_dz_st, dz, false, V, rows, L.ldz, 64, 32));
    // K4: dU chunk = coef invT (softmax - onehot), bf16
    rl::EpiParams ep = {};
    ep.rows = rows;
    ep.cols = V;
    ep.inv_temperature = s->inv_temperature;
    ep.scale_log2 = s->inv_temperature * 1.4426950408889634f;
    ep.targets = targets + c0;
    ep.vocab_offset = s->vocab_offset;
    ep.lse = lse + c0;
    ep.coef = coef + c0;
    ep.invt_rows = s->inv_temperature_rows ? s->inv_temperature_rows + c0 : nullptr;
    if (phases & RL_BWD_DU)
      RL_TRY((launch_gemm<rl::EPI_DZ, false, false>(RL_K_DZ_GEMM, t_h_k, t_w_k, t_dz_st, rows, V, H, group_m_for(RL_K_DZ_GEMM, 16), ep, sms, st)));
    // K6: dW (+)= dU^T h
    if ((phases & RL_BWD_DW) && dw) {
      RL_TRY(make_map(&t_dz_mn, dz, false, V, rows, L.ldz, 64, 64));
      RL_TRY(make_map(&t_h_mn, hc, false, H, rows, H, 64, 64));
      rl::EpiParams e6 = {};
      e6.rows = V;
      e6.cols = H;
      if (dw_nvls) {
        set_nvls(e6, dw_nvls, dw);
        RL_TRY((launch_gemm<rl::EPI_F32_NVLS, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                            group_m_for(RL_K_DW_GEMM, 8), e6, sms, st)));
      } else if (c0 == 0 && !accumulate_dw) {
        RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows, group_m_for(RL_K_DW_GEMM, 8), e6, sms, st)));
      } else {
        RL_TRY((launch_gemm<rl::EPI_F32_ADD, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows, group_m_for(RL_K_DW_GEMM, 8), e6, sms, st)));
      }
    }
    // K5: dH chunk = dU W
    if ((phases & RL_BWD_DH) && (dh || dh32)) {
      RL_TRY(make_map(&t_dz_k, dz, false, V, rows, L.ldz, 64, kARows));
      rl::EpiParams e5 = {};
      e5.rows = rows;
      e5.cols = H;
      if (dh) {
        RL_TRY(make_map(&t_dh, dh + c0 * H, false, H, rows, H, 64, 32));
        RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V, group_m_for(RL_K_DH_GEMM, 8), e5, sms, st)));
      } else {
        RL_TRY(make_map(&t_dh, dh32 + c0 * H, true, H, rows, H, 32, 32));
        if (dh_nvls) {
          set_nvls(e5, dh_nvls, dh32 + c0 * H);
          RL_TRY((launch_gemm<rl::EPI_F32_NVLS, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                               group_m_for(RL_K_DH_GEMM, 8), e5, sms, st)));
        } else
        RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V, group_m_for(RL_K_DH_GEMM, 8), e5, sms, st)));
      }
    }
  }
  return RL_OK;
}

// ------------------------------------------------------- Newton-Schulz (f3)
struct NsLayout {
  size_t xa, xb, g32, g16, g2, c16, parts, partials, sync, u, o, end;
  int64_t K;
  int splits;  // split-K of the Gram GEMM (its K x K output has few tiles)
};
constexpr int kNsMaxSplits = 8;
constexpr int kNsPartials = 1184;

NsLayout ns_layout(int64_t M, int64_t N, bool muon) {
  NsLayout l;
  Carve c;
  const int64_t K = M < N ? M : N;
  l.K = K;
  l.xa = c.take(static_cast<size_t>(M) * N * 2);
  l.xb = c.take(static_cast<size_t>(M) * N * 2);
  l.g32 = c.take(static_cast<size_t>(K) * K * 4);
  l.g16 = c.take(static_cast<size_t>(K) * K * 2);
  l.g2 = c.take(static_cast<size_t>(K) * K * 4);
  l.c16 = c.take(static_cast<size_t>(K) * K * 2);
  // splits: enough Gram tiles for >= 8 waves of CTA pairs, each split >= 64 k-blocks
  const int64_t tiles = ((K + 255) / 256) * ((K + 255) / 256);
  const int64_t kdim = M < N ? N : M;
  int sp = static_cast<int>((8 * 74 + tiles - 1) / tiles);
  while (sp > 1 && (kdim / 64) / sp < 64) --sp;
  l.splits = sp < 1 ? 1 : (sp > kNsMaxSplits ? kNsMaxSplits : sp);
  l.parts = c.take(static_cast<size_t>(l.splits) * K * K * 4);
  l.partials = c.take(kNsPartials * 8);
  l.sync = c.take(static_cast<size_t>(kMaxSyncPoints) * 4);
  l.u = muon ? c.take(static_cast<size_t>(M) * N * 4) : 0;
  l.o = muon ? c.take(static_cast<size_t>(M) * N * 2) : 0;
  l.end = align_up(c.off, 1024);
  return l;
}

rl_status check_ns_shape(int64_t M, int64_t N, int32_t steps) {
  if (M < 1 || N < 1 || M > (int64_t(1) << 31) - 1 || N > 65536) return fail(RL_ERR_SHAPE, "need 1 <= M and 1 <= N <= 65536");
  const int64_t K = M < N ? M : N;
  if (N % 8 != 0 || K % 8 != 0) return fail(RL_ERR_SHAPE, "N and min(M, N) must be multiples of 8");
  if (K > 16384) return fail(RL_ERR_SHAPE, "min(M, N) > 16384 (the K x K Gram would not fit the design)");
  if (steps < 1) return fail(RL_ERR_INVALID_ARGUMENT, "steps must be >= 1");
  return RL_OK;
}

// X_0 from g (fp32) in l.xa, then `steps` iterations; the last one writes `out`.
rl_status ns_impl(const float* g, int64_t M, int64_t N, int32_t steps, uint16_t* out, uint8_t* ws, const NsLayout& l,
                  int sms, cudaStream_t st) {
  constexpr float ca = 3.4445f, cb = -4.7750f, cc = 2.0315f;
  const int64_t K = l.K, n = M * N;
  const bool tall = M >= N;
  uint16_t* xa = reinterpret_cast<uint16_t*>(ws + l.xa);
  uint16_t* xb = reinterpret_cast<uint16_t*>(ws + l.xb);
  float* g32 = reinterpret_cast<float*>(ws + l.g32);
  uint16_t* g16 = reinterpret_cast<uint16_t*>(ws + l.g16);
  float* g2 = reinterpret_cast<float*>(ws + l.g2);
  uint16_t* c16 = reinterpret_cast<uint16_t*>(ws + l.c16);
  double* partials = reinterpret_cast<double*>(ws + l.partials);
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + l.sync);
  const int eblocks = 8 * sms;
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::sumsq_partial_kernel<<<kNsPartials, 256, 0, st>>>(g, n, partials);
  }
  RL_CHECK_LAUNCH();
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::ns_prep_kernel<<<eblocks, 256, 0, st>>>(g, n, partials, kNsPartials, xa);
  }
  RL_CHECK_LAUNCH();
  float* parts = reinterpret_cast<float*>(ws + l.parts);
  CUtensorMap t_g32, t_g16k, t_g16m, t_g2, t_c16m, t_c16k;
  RL_TRY(make_map(&t_g32, parts, true, K, K * l.splits, K, 32, 32));   // split s -> rows [s K, s K + K)
  RL_TRY(make_map(&t_g16k, g16, false, K, K, K, 64, kARows));
  RL_TRY(make_map(&t_g16m, g16, false, K, K, K, 64, 64));
  RL_TRY(make_map(&t_g2, g2, true, K, K, K, 32, 32));
  RL_TRY(make_map(&t_c16m, c16, false, K, K, K, 64, 64));
  RL_TRY(make_map(&t_c16k, c16, false, K, K, K, 64, kARows));
  rl::EpiParams e = {};
  uint16_t* src = xa;
  for (int j = 0; j < steps; ++j) {
    uint16_t* dst = (j == steps - 1) ? out : (src == xa ? xb : xa);
    CUtensorMap t_xk, t_xm, t_xb, t_out;
    RL_TRY(make_map(&t_xk, src, false, N, M, N, 64, kARows));          // X K-major (rows of X)
    RL_TRY(make_map(&t_xm, src, false, N, M, N, 64, 64));              // X MN-major
    RL_TRY(make_map(&t_xb, src, false, N, M, N, 64, rl::BN / cta_group()));  // X as a K-major B
    RL_TRY(make_map(&t_out, dst, false, N, M, N, 64, 32));
    e.rows = K;
    e.cols = K;
    if (tall) {  // A = X^T X : [N x N], K-dim = M
      RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_NS_GEMM, t_xm, t_xm, t_g32, N, N, M, 8, e, sms, st,
                                                   l.splits, static_cast<int>(K))));
    } else {     // A = X X^T : [M x M], K-dim = N
      RL_TRY((launch_gemm<rl::EPI_F32, false, false>(RL_K_NS_GEMM, t_xk, t_xb, t_g32, M, M, N, 8, e, sms, st,
                                                     l.splits, static_cast<int>(K))));
    }
    {
      ProfScope ps(RL_K_NS_AUX, st);
      rl::split_reduce_cast_kernel<<<eblocks, 256, 0, st>>>(parts, l.splits, K * K, g32, g16);
    }
    RL_CHECK_LAUNCH();
    RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_NS_GEMM, t_g16k, t_g16m, t_g2, K, K, K, 8, e, sms, st)));
    {
      ProfScope ps(RL_K_NS_AUX, st);
      rl::ns_poly_kernel<<<eblocks, 256, 0, st>>>(g32, g2, K, ca, cb, cc, c16);
    }
    RL_CHECK_LAUNCH();
    e.rows = M;
    e.cols = N;
    if (tall) {  // X' = X C : [M x N], K-dim = N
      RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_NS_GEMM, t_xk, t_c16m, t_out, M, N, N, 8, e, sms, st)));
    } else {     // X' = C X : [M x N], K-dim = M
      RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_NS_GEMM, t_c16k, t_xm, t_out, M, N, M, 8, e, sms, st)));
    }
    src = dst;
  }
  return RL_OK;
}

// Side stream + events of the host-I/O call (per host thread and device).
struct HostioStreams {
  int dev = -1;
  cudaStream_t copy = nullptr;
  cudaEvent_t start = nullptr, small = nullptr;
  std::vector<cudaEvent_t> slab;
  rl_status ensure(int n) {
    int d = 0;
    RL_CUDA(cudaGetDevice(&d));
    if (d != dev) {
      copy = nullptr;
      start = nullptr;
      small = nullptr;
      slab.clear();
      dev = d;
    }
    if (!copy) RL_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    if (!start) RL_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    if (!small) RL_CUDA(cudaEventCreateWithFlags(&small, cudaEventDisableTiming));
    while (static_cast<int>(slab.size()) < n) {
      cudaEvent_t e;
      RL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      slab.push_back(e);
    }
    return RL_OK;
  }
};
HostioStreams& hostio_streams() {
  thread_local HostioStreams h;
  return h;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* rl_status_string(rl_status s) {
  switch (s) {
    case RL_OK: return "RL_OK";
    case RL_ERR_INVALID_ARGUMENT: return "RL_ERR_INVALID_ARGUMENT";
    case RL_ERR_SHAPE: return "RL_ERR_SHAPE";
    case RL_ERR_UNSUPPORTED: return "RL_ERR_UNSUPPORTED";
    case RL_ERR_CUDA: return "RL_ERR_CUDA";
    case RL_ERR_WORKSPACE: return "RL_ERR_WORKSPACE";
    case RL_ERR_ALIGNMENT: return "RL_ERR_ALIGNMENT";
  }
  return "RL_ERR_UNKNOWN";
}

const char* rl_last_error_message(void) { return g_err; }
int32_t rl_abi_version(void) { return RL_ABI_VERSION; }
int32_t rl_last_launch_count(void) { return g_launches; }

rl_status rl_profile_enable(int32_t enable) {
  g_prof = enable != 0;
  return RL_OK;
}

int32_t rl_profile_read(rl_kernel_time* out, int32_t cap) {
  const int32_t n = static_cast<int32_t>(g_prof_recs.size());
  for (int32_t i = 0; i < n; ++i) {
    ProfRec& r = g_prof_recs[i];
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (out && i < cap) out[i] = rl_kernel_time{r.kernel, ms};
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  return n;
}

int64_t rl_default_dz_chunk_rows(const rl_lm_shape* shape) { return shape ? shape->T : 0; }

int64_t rl_nvls_flag_count(const rl_lm_shape* shape, int32_t which) {
  if (!shape) return 0;
  // slabs = tiles x 8 (2 CTAs x 4 epilogue warps), counted with the smaller
  // (128-row) tiles so the bound holds for either CTA-group variant
  const int64_t M = which == 0 ? shape->V_local : shape->T;
  return ((M + 127) / 128) * ((shape->H + rl::BN - 1) / rl::BN) * 8;
}

size_t rl_workspace_bytes(const rl_lm_shape* shape, int32_t num_rollouts, int64_t dz_chunk_rows) {
  if (check_shape(shape) != RL_OK) return 0;
  return ws_layout(shape, num_rollouts, dz_chunk_rows).end;
}

size_t rl_workspace_bytes_hostio(const rl_lm_shape* shape, int32_t num_rollouts, int64_t dz_chunk_rows) {
  if (check_shape(shape) != RL_OK) return 0;
  const size_t base = ws_layout(shape, num_rollouts, dz_chunk_rows).end;
  Carve c;
  c.off = base;
  const size_t T = static_cast<size_t>(shape->T), R = static_cast<size_t>(num_rollouts > 0 ? num_rollouts : 1);
  c.take(T * shape->H * 2);  // hidden
  c.take(T * 4);             // targets
  c.take(T * 4);             // infer
  c.take(R * 4);             // rewards
  c.take(R * 4);             // advantages
  c.take((R + 1) * 4);       // offsets
  c.take(T);                 // loss mask
  c.take(T * 4);             // logprob
  return align_up(c.off, 1024);
}

rl_status rl_group_advantages(const float* rewards, int32_t num_groups, int32_t group_size, float* advantages,
                              void* stream) {
  g_launches = 0;
  RL_NONNULL(rewards);
  RL_NONNULL(advantages);
  if (num_groups < 0) return fail(RL_ERR_SHAPE, "num_groups < 0");
  if (group_size < 2) return fail(RL_ERR_INVALID_ARGUMENT, "group_size must be >= 2 (got %d)", group_size);
  DevInfo d;
  RL_TRY(device_info(d));
  if (num_groups == 0) return RL_OK;
  const int threads = 256;
  const int blocks = static_cast<int>((static_cast<int64_t>(num_groups) * 32 + threads - 1) / threads);
  {
    ProfScope ps(RL_K_GROUP_ADV, static_cast<cudaStream_t>(stream));
    rl::group_adv_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(rewards, num_groups,
                                                                                    group_size, advantages);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_logprob_fwd(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                         const int32_t* targets, float* logprob, float* entropy, float* lse, void* workspace,
                         size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_TRY(check_shape(shape));
  if (shape->V_local != shape->V_global || shape->vocab_offset != 0)
    return fail(RL_ERR_SHAPE, "rl_logprob_fwd needs the full vocabulary; use rl_fwd_partials for a shard");
  if (shape->T > 0) {
    RL_NONNULL(hidden);
    RL_NONNULL(w_vocab);
    RL_NONNULL(targets);
    RL_NONNULL(logprob);
    if (!aligned16(hidden) || !aligned16(w_vocab) || !aligned16(workspace))
      return fail(RL_ERR_ALIGNMENT, "hidden, w_vocab and workspace must be 16-byte aligned");
  }
  const WsLayout L = ws_layout(shape, 1, 0);
  if (shape->T > 0 && (!workspace || workspace_bytes < L.dz))
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.dz, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  return forward_impl(shape, hidden, w_vocab, targets, logprob, entropy, lse, nullptr,
                      static_cast<uint8_t*>(workspace), L, d.sms, static_cast<cudaStream_t>(stream));
}

rl_status rl_fwd_partials(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                          const int32_t* targets, float* partials, void* workspace, size_t workspace_bytes,
                          void* stream) {
  g_launches = 0;
  RL_TRY(check_shape(shape));
  if (shape->T > 0) {
    RL_NONNULL(hidden);
    RL_NONNULL(w_vocab);
    RL_NONNULL(targets);
    RL_NONNULL(partials);
    if (!aligned16(hidden) || !aligned16(w_vocab) || !aligned16(workspace) || !aligned16(partials))
      return fail(RL_ERR_ALIGNMENT, "hidden, w_vocab, partials and workspace must be 16-byte aligned");
  }
  const WsLayout L = ws_layout(shape, 1, 0);
  if (shape->T > 0 && (!workspace || workspace_bytes < L.dz))
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.dz, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  return forward_impl(shape, hidden, w_vocab, targets, nullptr, nullptr, nullptr, reinterpret_cast<float4*>(partials),
                      static_cast<uint8_t*>(workspace), L, d.sms, static_cast<cudaStream_t>(stream));
}

rl_status rl_merge_partials(const float* partials, int32_t n_parts, int64_t T, float* logprob, float* entropy,
                            float* lse, void* stream) {
  g_launches = 0;
  if (T < 0 || n_parts < 1) return fail(RL_ERR_SHAPE, "need T >= 0 and n_parts >= 1");
  if (T == 0) return RL_OK;
  RL_NONNULL(partials);
  RL_NONNULL(logprob);
  if (!aligned16(partials)) return fail(RL_ERR_ALIGNMENT, "partials must be 16-byte aligned");
  DevInfo d;
  RL_TRY(device_info(d));
  const int blocks = static_cast<int>((T + rl::MERGE_ROWS - 1) / rl::MERGE_ROWS);
  {
    ProfScope ps(RL_K_MERGE, static_cast<cudaStream_t>(stream));
    rl::merge_partials_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const float4*>(partials), n_parts, T, logprob, entropy, lse, nullptr);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_loss_coef(const rl_loss_params* params, int64_t T, int64_t V_global, const float* logprob,
                       const float* infer_logprobs, const int32_t* targets, const float* rollout_adv,
                       const int32_t* rollout_offsets, const uint8_t* loss_mask, float* coef, uint8_t* token_keep,
                       uint8_t* rollout_guarded, rl_loss_report* report, void* workspace, size_t workspace_bytes,
                       void* stream) {
  g_launches = 0;
  RL_TRY(check_params(params));
  if (T < 0) return fail(RL_ERR_SHAPE, "T < 0");
  RL_NONNULL(rollout_adv);
  RL_NONNULL(rollout_offsets);
  RL_NONNULL(report);
  if (T > 0) {
    RL_NONNULL(logprob);
    RL_NONNULL(infer_logprobs);
    RL_NONNULL(coef);
  }
  const size_t need = static_cast<size_t>(params->num_rollouts) * sizeof(rl::RolloutPartial);
  if (!workspace || workspace_bytes < need)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  return loss_impl(params, T, V_global, logprob, infer_logprobs, targets, rollout_adv, rollout_offsets, loss_mask,
                   coef, token_keep, rollout_guarded, report, static_cast<rl::RolloutPartial*>(workspace),
                   static_cast<cudaStream_t>(stream));
}

rl_status rl_bwd(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab, const int32_t* targets,
                 const float* lse, const float* coef, uint16_t* d_hidden, float* d_hidden_f32, float* d_w_vocab,
                 int32_t accumulate_dw, int64_t dz_chunk_rows, void* workspace, size_t workspace_bytes,
                 void* stream) {
  return rl_bwd_ex(shape, hidden, w_vocab, targets, lse, coef, d_hidden, d_hidden_f32, d_w_vocab, accumulate_dw,
                   dz_chunk_rows, RL_BWD_ALL, 0, nullptr, nullptr, workspace, workspace_bytes, stream);
}

rl_status rl_bwd_ex(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                    const int32_t* targets, const float* lse, const float* coef, uint16_t* d_hidden,
                    float* d_hidden_f32, float* d_w_vocab, int32_t accumulate_dw, int64_t dz_chunk_rows,
                    int32_t phases, int32_t max_sms, const rl_nvls_reduce* dw_nvls,
                    const rl_nvls_reduce* dh_nvls, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_TRY(check_nvls(dw_nvls, "dw_nvls"));
  RL_TRY(check_nvls(dh_nvls, "dh_nvls"));
  if (dw_nvls && accumulate_dw) return fail(RL_ERR_INVALID_ARGUMENT, "dw_nvls needs accumulate_dw = 0");
  if (dh_nvls && !d_hidden_f32) return fail(RL_ERR_INVALID_ARGUMENT, "dh_nvls reduces d_hidden_f32");
  if ((phases & RL_BWD_ALL) == 0 || (phases & ~(RL_BWD_ALL | RL_BWD_DENSE)) != 0)
    return fail(RL_ERR_INVALID_ARGUMENT, "phases must be a non-empty RL_BWD_* mask");
  if (max_sms < 0) return fail(RL_ERR_INVALID_ARGUMENT, "max_sms must be >= 0");
  RL_TRY(check_shape(shape));
  if (d_hidden && d_hidden_f32) return fail(RL_ERR_INVALID_ARGUMENT, "pass d_hidden or d_hidden_f32, not both");
  RL_NONNULL(w_vocab);
  if (shape->T > 0) {
    RL_NONNULL(hidden);
    RL_NONNULL(targets);
    RL_NONNULL(lse);
    RL_NONNULL(coef);
  }
  if (!aligned16(hidden) || !aligned16(w_vocab) || !aligned16(workspace) || !aligned16(d_hidden) ||
      !aligned16(d_hidden_f32) || !aligned16(d_w_vocab))
    return fail(RL_ERR_ALIGNMENT, "matrix pointers and workspace must be 16-byte aligned");
  const WsLayout L = ws_layout(shape, 1, dz_chunk_rows);
  if (shape->T > 0 && (!workspace || workspace_bytes < L.end))
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.end, workspace_bytes);
  if ((phases & RL_BWD_ALL) != RL_BWD_ALL && L.chunk < shape->T)
    return fail(RL_ERR_INVALID_ARGUMENT, "partial backward phases need one dU chunk (dz_chunk_rows = 0 or >= T)");
  if ((dw_nvls || dh_nvls) && L.chunk < shape->T)
    return fail(RL_ERR_INVALID_ARGUMENT, "NVLS reduction needs one dU chunk (dz_chunk_rows = 0 or >= T)");
  DevInfo d;
  RL_TRY(device_info(d));
  int sms = d.sms;
  if (max_sms > 0 && max_sms < sms) sms = max_sms < 2 ? 2 : max_sms;
  return bwd_impl(shape, hidden, w_vocab, targets, lse, coef, d_hidden, d_hidden_f32, d_w_vocab, accumulate_dw,
                  static_cast<uint8_t*>(workspace), L, sms, static_cast<cudaStream_t>(stream), phases, dw_nvls,
                  dh_nvls);
}

// The whole step. With slab_events, the forward runs slab by slab (slab_rows
// rows each), each launch first waiting for its slab's event (the host-I/O
// call records one per H2D slab copy), so the hidden-state upload overlaps K1.
static rl_status step_impl(const rl_lm_shape* shape, const rl_loss_params* params, const uint16_t* hidden,
                           const uint16_t* w_vocab, const int32_t* targets, const float* infer_logprobs,
                           const float* rollout_adv, const int32_t* rollout_offsets, const uint8_t* loss_mask,
                           const rl_loss_outputs* out, uint8_t* ws, const WsLayout& L, int sms, cudaStream_t st,
                           const cudaEvent_t* slab_events = nullptr, const int64_t* slab_ends = nullptr) {
  float* lse = out->lse ? out->lse : reinterpret_cast<float*>(ws + L.lse);
  float* coef = out->coef ? out->coef : reinterpret_cast<float*>(ws + L.coef);
  if (slab_events && slab_ends && shape->T > 0) {
    int j = 0;
    for (int64_t r0 = 0; r0 < shape->T; r0 = slab_ends[j], ++j) {
      rl_lm_shape sub = *shape;
      sub.T = slab_ends[j] - r0;
      if (shape->inv_temperature_rows) sub.inv_temperature_rows = shape->inv_temperature_rows + r0;
      RL_CUDA(cudaStreamWaitEvent(st, slab_events[j], 0));
      RL_TRY(forward_impl(&sub, hidden + r0 * shape->H, w_vocab, targets + r0, out->logprob + r0,
                          out->entropy ? out->entropy + r0 : nullptr, lse + r0, nullptr, ws, L, sms, st));
    }
  } else {
    RL_TRY(forward_impl(shape, hidden, w_vocab, targets, out->logprob, out->entropy, lse, nullptr, ws, L, sms, st));
  }
  RL_TRY(loss_impl(params, shape->T, shape->V_global, out->logprob, infer_logprobs, targets, rollout_adv,
                   rollout_offsets, loss_mask, coef, out->token_keep, out->rollout_guarded, out->report,
                   reinterpret_cast<rl::RolloutPartial*>(ws + L.rp), st));
  RL_TRY(bwd_impl(shape, hidden, w_vocab, targets, lse, coef, out->d_hidden, out->d_hidden_f32, out->d_w_vocab,
                  out->accumulate_dw, ws, L, sms, st, RL_BWD_ALL | (out->dense_backward ? RL_BWD_DENSE : 0),
                  out->d_w_vocab_nvls, nullptr));
  return RL_OK;
}

static rl_status check_step_args(const rl_lm_shape* shape, const rl_loss_params* params, const uint16_t* w_vocab,
                                 const rl_loss_outputs* out, bool need_logprob) {
  RL_TRY(check_shape(shape));
  RL_TRY(check_params(params));
  if (shape->V_local != shape->V_global || shape->vocab_offset != 0)
    return fail(RL_ERR_SHAPE, "rl_policy_loss_fwd_bwd needs the full vocabulary; vocab-parallel callers use the split phases");
  RL_NONNULL(out);
  RL_NONNULL(out->report);
  RL_NONNULL(w_vocab);
  if (out->d_hidden && out->d_hidden_f32) return fail(RL_ERR_INVALID_ARGUMENT, "pass d_hidden or d_hidden_f32, not both");
  if (!aligned16(w_vocab) || !aligned16(out->d_hidden) || !aligned16(out->d_hidden_f32) || !aligned16(out->d_w_vocab))
    return fail(RL_ERR_ALIGNMENT, "matrix pointers must be 16-byte aligned");
  if (need_logprob && shape->T > 0) RL_NONNULL(out->logprob);
  RL_TRY(check_nvls(out->d_w_vocab_nvls, "d_w_vocab_nvls"));
  if (out->d_w_vocab_nvls && (out->accumulate_dw || !out->d_w_vocab))
    return fail(RL_ERR_INVALID_ARGUMENT, "d_w_vocab_nvls needs d_w_vocab and accumulate_dw = 0");
  if (out->dz_chunk_rows < 0) return fail(RL_ERR_INVALID_ARGUMENT, "dz_chunk_rows must be >= 0");
  if (out->d_w_vocab_nvls && out->dz_chunk_rows > 0 && out->dz_chunk_rows < shape->T)
    return fail(RL_ERR_INVALID_ARGUMENT, "d_w_vocab_nvls needs one dU chunk (dz_chunk_rows = 0 or >= T)");
  return RL_OK;
}

rl_status rl_policy_loss_fwd_bwd(const rl_lm_shape* shape, const rl_loss_params* params, const uint16_t* hidden,
                                 const uint16_t* w_vocab, const int32_t* targets, const float* infer_logprobs,
                                 const float* rollout_adv, const int32_t* rollout_offsets, const uint8_t* loss_mask,
                                 const rl_loss_outputs* out, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_TRY(check_step_args(shape, params, w_vocab, out, true));
  RL_NONNULL(rollout_adv);
  RL_NONNULL(rollout_offsets);
  if (shape->T > 0) {
    RL_NONNULL(hidden);
    RL_NONNULL(targets);
    RL_NONNULL(infer_logprobs);
    if (!aligned16(hidden)) return fail(RL_ERR_ALIGNMENT, "hidden must be 16-byte aligned");
  }
  const WsLayout L = ws_layout(shape, params->num_rollouts, out->dz_chunk_rows);
  if (!workspace || workspace_bytes < L.end)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.end, workspace_bytes);
  if (!aligned16(workspace)) return fail(RL_ERR_ALIGNMENT, "workspace must be 16-byte aligned");
  DevInfo d;
  RL_TRY(device_info(d));
  return step_impl(shape, params, hidden, w_vocab, targets, infer_logprobs, rollout_adv, rollout_offsets, loss_mask,
                   out, static_cast<uint8_t*>(workspace), L, d.sms, static_cast<cudaStream_t>(stream));
}

rl_status rl_policy_loss_fwd_bwd_hostio(const rl_lm_shape* shape, const rl_loss_params* params, int32_t group_size,
                                        const uint16_t* hidden_host, const uint16_t* w_vocab,
                                        const int32_t* targets_host, const float* infer_host,
                                        const float* rewards_host, const int32_t* offsets_host,
                                        const uint8_t* loss_mask_host, const rl_loss_outputs* out,
                                        rl_loss_report* report_host, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  g_launches = 0;
  RL_TRY(check_step_args(shape, params, w_vocab, out, false));
  RL_NONNULL(rewards_host);
  RL_NONNULL(offsets_host);
  RL_NONNULL(report_host);
  if (group_size < 2 || params->num_rollouts % group_size != 0)
    return fail(RL_ERR_INVALID_ARGUMENT, "group_size must be >= 2 and divide num_rollouts");
  const int64_t T = shape->T;
  if (T > 0) {
    RL_NONNULL(hidden_host);
    RL_NONNULL(targets_host);
    RL_NONNULL(infer_host);
  }
  const size_t need = rl_workspace_bytes_hostio(shape, params->num_rollouts, out->dz_chunk_rows);
  if (!workspace || workspace_bytes < need)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  if (!aligned16(workspace)) return fail(RL_ERR_ALIGNMENT, "workspace must be 16-byte aligned");
  DevInfo d;
  RL_TRY(device_info(d));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const WsLayout L = ws_layout(shape, params->num_rollouts, out->dz_chunk_rows);
  Carve c;
  c.off = L.end;
  const size_t R = static_cast<size_t>(params->num_rollouts);
  uint16_t* d_hidden_in = reinterpret_cast<uint16_t*>(ws + c.take(T * shape->H * 2));
  int32_t* d_tg = reinterpret_cast<int32_t*>(ws + c.take(T * 4));
  float* d_inf = reinterpret_cast<float*>(ws + c.take(T * 4));
  float* d_rw = reinterpret_cast<float*>(ws + c.take(R * 4));
  float* d_adv = reinterpret_cast<float*>(ws + c.take(R * 4));
  int32_t* d_off = reinterpret_cast<int32_t*>(ws + c.take((R + 1) * 4));
  uint8_t* d_lm = ws + c.take(T);
  float* d_lp = reinterpret_cast<float*>(ws + c.take(T * 4));
  // hidden rows go up in slabs on a side stream; the forward starts on slab 0
  // while the rest is in flight (the small per-token vectors go first on `st`)
  // slab ends: 1024, 4096, then every 4096 rows (a small first slab shortens the
  // exposed part of the upload; later slabs keep the forward's tiles large)
  std::vector<int64_t> ends;
  for (int64_t e = 1024; ; e = (e < 4096) ? 4096 : e + 4096) {
    ends.push_back(e < T ? e : T);
    if (e >= T) break;
  }
  const int n_slabs = static_cast<int>(ends.size());
  HostioStreams& hs = hostio_streams();
  RL_TRY(hs.ensure(n_slabs));
  // every upload goes through the copy stream, in the order the compute needs it:
  // the small per-token/per-rollout vectors first (event `small`), then the
  // hidden-state slabs (one event each); H2D copies share the copy engine's FIFO,
  // so nothing the first kernels need may queue behind the big slabs
  RL_CUDA(cudaEventRecord(hs.start, st));
  RL_CUDA(cudaStreamWaitEvent(hs.copy, hs.start, 0));
  if (T > 0) {
    RL_CUDA(cudaMemcpyAsync(d_tg, targets_host, T * 4, cudaMemcpyHostToDevice, hs.copy));
    RL_CUDA(cudaMemcpyAsync(d_inf, infer_host, T * 4, cudaMemcpyHostToDevice, hs.copy));
    if (loss_mask_host) RL_CUDA(cudaMemcpyAsync(d_lm, loss_mask_host, T, cudaMemcpyHostToDevice, hs.copy));
  }
  RL_CUDA(cudaMemcpyAsync(d_rw, rewards_host, R * 4, cudaMemcpyHostToDevice, hs.copy));
  RL_CUDA(cudaMemcpyAsync(d_off, offsets_host, (R + 1) * 4, cudaMemcpyHostToDevice, hs.copy));
  RL_CUDA(cudaEventRecord(hs.small, hs.copy));
  for (int j = 0; T > 0 && j < n_slabs; ++j) {
    const int64_t r0 = j == 0 ? 0 : ends[j - 1], rows = ends[j] - r0;
    RL_CUDA(cudaMemcpyAsync(d_hidden_in + r0 * shape->H, hidden_host + r0 * shape->H, rows * shape->H * 2,
                            cudaMemcpyHostToDevice, hs.copy));
    RL_CUDA(cudaEventRecord(hs.slab[j], hs.copy));
  }
  RL_CUDA(cudaStreamWaitEvent(st, hs.small, 0));
  const int ng = static_cast<int>(R / group_size);
  {
    ProfScope ps(RL_K_GROUP_ADV, st);
    rl::group_adv_kernel<<<(ng * 32 + 255) / 256, 256, 0, st>>>(d_rw, ng, group_size, d_adv);
  }
  RL_CHECK_LAUNCH();
  rl_loss_outputs o = *out;
  if (!o.logprob) o.logprob = d_lp;
  rl_status s = step_impl(shape, params, d_hidden_in, w_vocab, d_tg, d_inf, d_adv, d_off,
                          loss_mask_host ? d_lm : nullptr, &o, ws, L, d.sms, st, T > 0 ? hs.slab.data() : nullptr,
                          T > 0 ? ends.data() : nullptr);
  if (s != RL_OK) return s;
  RL_CUDA(cudaMemcpyAsync(report_host, out->report, sizeof(rl_loss_report), cudaMemcpyDeviceToHost, st));
  RL_CUDA(cudaStreamSynchronize(st));
  return RL_OK;
}

rl_status rl_rms_inv(const uint16_t* x, int64_t rows, int64_t K, float eps, float* out, void* stream) {
  g_launches = 0;
  if (rows < 0 || K < 1) return fail(RL_ERR_SHAPE, "need rows >= 0 and K >= 1");
  if (!(eps >= 0.f) || !isfinite(eps)) return fail(RL_ERR_INVALID_ARGUMENT, "eps must be finite and >= 0");
  if (rows == 0) return RL_OK;
  RL_NONNULL(x);
  RL_NONNULL(out);
  DevInfo d;
  RL_TRY(device_info(d));
  const int64_t threads = rows * 32;
  {
    ProfScope ps(RL_K_NS_AUX, static_cast<cudaStream_t>(stream));
    rl::rms_inv_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, rows, K, eps, out);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

size_t rl_newton_schulz_workspace_bytes(int64_t M, int64_t N) {
  if (check_ns_shape(M, N, 1) != RL_OK) return 0;
  return ns_layout(M, N, false).end;
}

size_t rl_muon_workspace_bytes(int64_t M, int64_t N) {
  if (check_ns_shape(M, N, 1) != RL_OK) return 0;
  return ns_layout(M, N, true).end;
}

rl_status rl_newton_schulz(const float* g, int64_t M, int64_t N, int32_t steps, uint16_t* out, void* workspace,
                           size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_TRY(check_ns_shape(M, N, steps));
  RL_NONNULL(g);
  RL_NONNULL(out);
  if (!aligned16(g) || !aligned16(out) || !aligned16(workspace))
    return fail(RL_ERR_ALIGNMENT, "g, out and workspace must be 16-byte aligned");
  const NsLayout l = ns_layout(M, N, false);
  if (!workspace || workspace_bytes < l.end)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", l.end, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  return ns_impl(g, M, N, steps, out, static_cast<uint8_t*>(workspace), l, d.sms, static_cast<cudaStream_t>(stream));
}

rl_status rl_muon_step(float* theta, const float* grad, float* momentum, int64_t M, int64_t N, float lr, float mu,
                       float weight_decay, int32_t nesterov, int32_t steps, void* workspace, size_t workspace_bytes,
                       void* stream) {
  g_launches = 0;
  RL_TRY(check_ns_shape(M, N, steps));
  RL_NONNULL(theta);
  RL_NONNULL(grad);
  RL_NONNULL(momentum);
  if (!aligned16(theta) || !aligned16(grad) || !aligned16(momentum) || !aligned16(workspace))
    return fail(RL_ERR_ALIGNMENT, "theta, grad, momentum and workspace must be 16-byte aligned");
  if (!isfinite(lr) || !isfinite(mu) || !isfinite(weight_decay))
    return fail(RL_ERR_INVALID_ARGUMENT, "lr, mu and weight_decay must be finite");
  const NsLayout l = ns_layout(M, N, true);
  if (!workspace || workspace_bytes < l.end)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", l.end, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  float* u = reinterpret_cast<float*>(ws + l.u);
  uint16_t* o = reinterpret_cast<uint16_t*>(ws + l.o);
  const int64_t n = M * N;
  const int eblocks = 4 * d.sms;
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::muon_momentum_kernel<<<eblocks, 256, 0, st>>>(grad, momentum, u, n, mu, nesterov ? 1 : 0);
  }
  RL_CHECK_LAUNCH();
  RL_TRY(ns_impl(u, M, N, steps, o, ws, l, d.sms, st));
  const double scale = sqrt(M > N ? static_cast<double>(M) / N : 1.0);
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::muon_apply_kernel<<<eblocks, 256, 0, st>>>(theta, o, n, 1.f - lr * weight_decay,
                                                   static_cast<float>(lr * scale));
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}


rl_status rl_grouped_gemm(const uint16_t* a, const uint16_t* b, const int32_t* offsets, int32_t n_groups, int64_t rows,
                          int64_t N, int64_t K, const float* row_scale, uint16_t* out, void* stream) {
  g_launches = 0;
  if (n_groups < 1 || n_groups > rl::MAX_GROUPS) return fail(RL_ERR_SHAPE, "need 1 <= n_groups <= %d", rl::MAX_GROUPS);
  if (rows < 0 || rows > (int64_t(1) << 31) - 1 || N < 32 || N % 32 != 0 || K < 8 || K % 8 != 0 ||
      static_cast<int64_t>(n_groups) * N > (int64_t(1) << 31) - 1)
    return fail(RL_ERR_SHAPE, "need rows >= 0, N a positive multiple of 32, K a positive multiple of 8");
  if (rows == 0) return RL_OK;
  RL_NONNULL(a);
  RL_NONNULL(b);
  RL_NONNULL(offsets);
  RL_NONNULL(out);
  if (!aligned16(a) || !aligned16(b) || !aligned16(out)) return fail(RL_ERR_ALIGNMENT, "a, b and out must be 16-byte aligned");
  DevInfo d;
  RL_TRY(device_info(d));
  CUtensorMap ta, tb, tc;
  RL_TRY(make_map(&ta, a, false, K, rows, K, 64, kARows));
  RL_TRY(make_map(&tb, b, false, K, static_cast<int64_t>(n_groups) * N, K, 64, rl::BN / cta_group()));
  RL_TRY(make_map(&tc, out, false, N, rows, N, 64, 32));
  rl::EpiParams ep = {};
  ep.rows = rows;
  ep.cols = N;
  ep.group_offsets = offsets;
  ep.n_groups = n_groups;
  ep.grouped_out = out;
  ep.row_scale = row_scale;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cta_group() == 2) return launch_grouped_cg<2>(ta, tb, tc, rows, N, K, n_groups, ep, d.sms, st);
  return launch_grouped_cg<1>(ta, tb, tc, rows, N, K, n_groups, ep, d.sms, st);
}

}  // extern "C"

// Diagnostics (not part of rl.h): how many clusters of `cluster` CTAs of the
// forward GEMM (CG=2 smem footprint) can be co-resident on this device.
extern "C" int32_t rl_debug_max_active_clusters(int32_t cluster) {
  auto kern = rl::gemm_kernel<rl::EPI_LSE, false, false, 2, 6>;
  constexpr int smem = rl::gemm_smem_bytes<2, 6>();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
  if (cluster > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = dim3(rl::GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return -2;
  return n;
}
