// librl host code: Newton-Schulz / Muon driver and the host-I/O copy stream.
// Included once, in order, by rl_api.cu (a single translation unit); everything
// here has internal linkage.
#pragma once

namespace {

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
      RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_NS_GEMM, t_xm, t_xm, t_g32, N, N, M, group_m_for(RL_K_NS_GEMM, 8), e, sms, st,
                                                   l.splits, static_cast<int>(K))));
    } else {     // A = X X^T : [M x M], K-dim = N
      RL_TRY((launch_gemm<rl::EPI_F32, false, false>(RL_K_NS_GEMM, t_xk, t_xb, t_g32, M, M, N, group_m_for(RL_K_NS_GEMM, 8), e, sms, st,
                                                     l.splits, static_cast<int>(K))));
    }
    {
      ProfScope ps(RL_K_NS_AUX, st);
      rl::split_reduce_cast_kernel<<<eblocks, 256, 0, st>>>(parts, l.splits, K * K, g32, g16);
    }
    RL_CHECK_LAUNCH();
    RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_NS_GEMM, t_g16k, t_g16m, t_g2, K, K, K, group_m_for(RL_K_NS_GEMM, 8), e, sms, st)));
    {
      ProfScope ps(RL_K_NS_AUX, st);
      rl::ns_poly_kernel<<<eblocks, 256, 0, st>>>(g32, g2, K, ca, cb, cc, c16);
    }
    RL_CHECK_LAUNCH();
    e.rows = M;
    e.cols = N;
    if (tall) {  // X' = X C : [M x N], K-dim = N
      RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_NS_GEMM, t_xk, t_c16m, t_out, M, N, N, group_m_for(RL_K_NS_GEMM, 8), e, sms, st)));
    } else {     // X' = C X : [M x N], K-dim = M
      RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_NS_GEMM, t_c16k, t_xm, t_out, M, N, M, group_m_for(RL_K_NS_GEMM, 8), e, sms, st)));
    }
    src = dst;
  }
  return RL_OK;
}

// Row-sharded Newton-Schulz (tall): the phases of ns_impl between which the caller
// all-reduces the sum of squares and the Gram. X_j lives in xa (j even) / xb (j odd).
rl_status ns_shard_sumsq_impl(const float* g, int64_t M, int64_t N, double* sumsq, uint8_t* ws, const NsLayout& l,
                              cudaStream_t st) {
  double* partials = reinterpret_cast<double*>(ws + l.partials);
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::sumsq_partial_kernel<<<kNsPartials, 256, 0, st>>>(g, M * N, partials);
  }
  RL_CHECK_LAUNCH();
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::sum_partials_kernel<<<1, 256, 0, st>>>(partials, kNsPartials, sumsq);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status ns_shard_gram_impl(int j, const float* g, const double* sumsq, int64_t M, int64_t N, float* gram, uint8_t* ws,
                             const NsLayout& l, int sms, cudaStream_t st) {
  const int64_t K = l.K;  // = N (tall shard)
  uint16_t* xa = reinterpret_cast<uint16_t*>(ws + l.xa);
  uint16_t* xb = reinterpret_cast<uint16_t*>(ws + l.xb);
  uint16_t* g16 = reinterpret_cast<uint16_t*>(ws + l.g16);
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + l.sync);
  if (j == 0) {
    ProfScope ps(RL_K_NS_AUX, st);
    // the global sum of squares as a single "partial": every block reads the same value
    rl::ns_prep_kernel<<<8 * sms, 256, 0, st>>>(g, M * N, sumsq, 1, xa);
  }
  RL_CHECK_LAUNCH();
  uint16_t* src = (j % 2 == 0) ? xa : xb;
  float* parts = reinterpret_cast<float*>(ws + l.parts);
  CUtensorMap t_xm, t_g32;
  RL_TRY(make_map(&t_xm, src, false, N, M, N, 64, 64));
  RL_TRY(make_map(&t_g32, parts, true, K, K * l.splits, K, 32, 32));
  rl::EpiParams e = {};
  e.rows = K;
  e.cols = K;
  RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_NS_GEMM, t_xm, t_xm, t_g32, N, N, M, group_m_for(RL_K_NS_GEMM, 8), e, sms, st, l.splits,
                                               static_cast<int>(K))));
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::split_reduce_cast_kernel<<<8 * sms, 256, 0, st>>>(parts, l.splits, K * K, gram, g16);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status ns_shard_apply_impl(int j, int steps, const float* gram, int64_t M, int64_t N, uint16_t* out, uint8_t* ws,
                              const NsLayout& l, int sms, cudaStream_t st) {
  constexpr float ca = 3.4445f, cb = -4.7750f, cc = 2.0315f;
  const int64_t K = l.K;
  uint16_t* xa = reinterpret_cast<uint16_t*>(ws + l.xa);
  uint16_t* xb = reinterpret_cast<uint16_t*>(ws + l.xb);
  uint16_t* g16 = reinterpret_cast<uint16_t*>(ws + l.g16);
  float* g2 = reinterpret_cast<float*>(ws + l.g2);
  uint16_t* c16 = reinterpret_cast<uint16_t*>(ws + l.c16);
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + l.sync);
  uint16_t* src = (j % 2 == 0) ? xa : xb;
  uint16_t* dst = (j == steps - 1) ? out : ((j % 2 == 0) ? xb : xa);
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::cast_bf16_kernel<<<8 * sms, 256, 0, st>>>(gram, K * K, g16);   // the all-reduced Gram
  }
  RL_CHECK_LAUNCH();
  CUtensorMap t_g16k, t_g16m, t_g2, t_c16m, t_xk, t_out;
  RL_TRY(make_map(&t_g16k, g16, false, K, K, K, 64, kARows));
  RL_TRY(make_map(&t_g16m, g16, false, K, K, K, 64, 64));
  RL_TRY(make_map(&t_g2, g2, true, K, K, K, 32, 32));
  RL_TRY(make_map(&t_c16m, c16, false, K, K, K, 64, 64));
  RL_TRY(make_map(&t_xk, src, false, N, M, N, 64, kARows));
  RL_TRY(make_map(&t_out, dst, false, N, M, N, 64, 32));
  rl::EpiParams e = {};
  e.rows = K;
  e.cols = K;
  RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_NS_GEMM, t_g16k, t_g16m, t_g2, K, K, K, group_m_for(RL_K_NS_GEMM, 8), e, sms, st)));
  {
    ProfScope ps(RL_K_NS_AUX, st);
    rl::ns_poly_kernel<<<8 * sms, 256, 0, st>>>(gram, g2, K, ca, cb, cc, c16);
  }
  RL_CHECK_LAUNCH();
  e.rows = M;
  e.cols = N;
  RL_TRY((launch_gemm<rl::EPI_BF16, false, true>(RL_K_NS_GEMM, t_xk, t_c16m, t_out, M, N, N, group_m_for(RL_K_NS_GEMM, 8), e, sms, st)));
  return RL_OK;
}

// Side stream + events of the host-I/O call, one set per host thread and device
// (streams and events belong to the device that was current when they were made,
// so a thread that switches devices gets another set instead of dropping this one).
struct HostioStreams {
  cudaStream_t copy = nullptr;
  cudaEvent_t start = nullptr, small = nullptr;
  std::vector<cudaEvent_t> slab;
  rl_status ensure(int n) {
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
constexpr int kMaxDevices = 64;
rl_status hostio_streams(HostioStreams*& out) {
  thread_local std::array<HostioStreams, kMaxDevices> per_device;
  int d = 0;
  RL_CUDA(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) return fail(RL_ERR_UNSUPPORTED, "device index %d out of range", d);
  out = &per_device[d];
  return RL_OK;
}

}  // namespace
