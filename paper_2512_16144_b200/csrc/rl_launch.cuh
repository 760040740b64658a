// librl host code: TMA tensor maps, the tuning knobs (CTA group, raster, soft k-barrier, wide tiles) and the GEMM launchers.
// Included once, in order, by rl_api.cu (a single translation unit); everything
// here has internal linkage.
#pragma once

namespace {

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
                   int box_inner, int box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
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
                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(RL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for [%lld x %lld] box %dx%d", (int)r,
                (long long)outer, (long long)inner, box_outer, box_inner);
  return RL_OK;
}

// ----------------------------------------------------------------- GEMMs
// Tuning knobs are read from the environment once per process, in thread-safe
// static initialisers (C++11 magic statics), and never change afterwards.

// CTA-pair (cta_group::2, 256x256 tiles) by default; RL_CTA_GROUP=1 selects the
// single-CTA 128x256 variant (kept for A/B measurements and as a fallback).
int cta_group() {
  static const int cg = [] {
    const char* e = getenv("RL_CTA_GROUP");
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return cg;
}

// Raster group of the wide dH / dW GEMMs: tiles walk n inside groups of 2 m-blocks.
// DRAM reads per launch at GLM-16k: 8 -> 17.3 GB, 4 -> 15.6, 2 -> 14.7; step -0.8 ms
// (profiles/r01/raster_traffic/, bwd_group_ab/).
constexpr int kGroupMBwd = 2;

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
constexpr int kKnobKids = 32;
// getenv("<base>_<K>"), else getenv("<base>"), else `unset`, for every kernel id
std::array<int, kKnobKids> env_table(const char* base, int unset) {
  std::array<int, kKnobKids> t;
  for (int kid = 0; kid < kKnobKids; ++kid) {
    char name[64];
    snprintf(name, sizeof(name), "%s_%s", base, kid_suffix(kid));
    const char* e = getenv(name);
    if (!e) e = getenv(base);
    t[kid] = e ? atoi(e) : unset;
  }
  return t;
}

// Raster group (in m-blocks) per GEMM: tiles walk n inside groups of this many
// m-blocks. Defaults chosen from the sweep in DESIGN.md §5 (passed by the call
// site); RL_GROUP_M_<K> (K in FWD, DZ, DH, DW, NS) overrides for measurements.
int group_m_for(int kid, int dflt) {
  static const std::array<int, kKnobKids> env = [] {
    std::array<int, kKnobKids> t;
    for (int kid = 0; kid < kKnobKids; ++kid) {
      char name[64];
      snprintf(name, sizeof(name), "RL_GROUP_M_%s", kid_suffix(kid));
      const char* e = getenv(name);
      t[kid] = e ? atoi(e) : 0;
    }
    return t;
  }();
  if (kid < 0 || kid >= kKnobKids) return dflt;
  return env[kid] > 0 ? env[kid] : dflt;
}

// Soft k-barrier between producers (see EpiParams::sync_*): every RL_SYNC_EVERY
// k-blocks (default 32, 16 for the wide dH/dW GEMMs; 0 = off), at most RL_SYNC_SLACK sync points of lead
// (default 2). Keeping the CTAs that share operands inside one L2 window cuts
// K5/K6 DRAM reads by ~1/3 and lets the power-capped clock rise (~6% per step,
// profiles/r01/). Correctness never depends on it (the wait is bounded).
// Per-GEMM overrides: RL_SYNC_EVERY_<K>, RL_SYNC_SLACK_<K> (K in FWD, DZ, DH, DW, NS).
int sync_every_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_SYNC_EVERY", -1);
  if (kid < 0 || kid >= kKnobKids) return 0;
  // 16 for the wide dH / dW GEMMs (their 48 KB k-blocks move twice the bytes per
  // window): DRAM reads 23.4 -> 17.3 GB each, step 60.7 -> 59.6 ms
  // (profiles/r01/sync_window_ab/); 32 elsewhere
  if (env[kid] >= 0) return env[kid];
  return (kid == RL_K_DH_GEMM || kid == RL_K_DW_GEMM) ? 16 : 32;
}
// Wide 256 x 512 pair tiles (NB = 2, rl_gemm.cuh): RL_WIDE[_<K>] = 0/1, default on
// for K1 (FWD), K5 (DH), K6 (DW) and the Newton-Schulz GEMMs (NS: 41.0 -> 38.6 ms); RL_SKEW = 0/2/3 k-blocks of block-0-first MMA
// order at both ends of a tile (default 3), which hides the epilogue of one TMEM
// half. K4 (DZ) stays narrow: its exp + bf16-store epilogue per half is longer
// than that cover (measured: K4 15.6 -> 17.9 ms wide, K1 15.6 -> 15.2 ms).
bool wide_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_WIDE", -1);
  if (kid < 0 || kid >= kKnobKids) return false;
  if (env[kid] >= 0) return env[kid] != 0;
  return kid == RL_K_FWD_GEMM || kid == RL_K_DH_GEMM || kid == RL_K_DW_GEMM || kid == RL_K_NS_GEMM;
}
// Serpentine K order (EpiParams::k_serpentine): the tiles of odd waves (tile / pairs odd)
// walk their k-blocks backwards. The CTAs of a wave run in k-lockstep (the soft k-barrier),
// so a wave starts on the operand rows the previous wave read last, which are still in L2: the dW GEMM re-reads hidden [T, H] once per wave (~64 waves at GLM-16k).
// RL_SERPENTINE[_<K>] = 0/1; default on for K6 (DW) and the Newton-Schulz GEMMs (the Gram
// re-reads X). Off for K5 (DH): its accumulation order per dH row would then depend on the
// wave the row lands in, and the sparse backward's dH is bitwise the dense one only while
// every tile sums in the same order; off for K1 / K4 (K = H, nothing to reuse).
bool serpentine_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_SERPENTINE", -1);
  if (kid < 0 || kid >= kKnobKids) return false;
  if (env[kid] >= 0) return env[kid] != 0;
  return kid == RL_K_DW_GEMM || kid == RL_K_NS_GEMM;
}
// Dynamic tile order (EpiParams::dyn_tiles): RL_DYN_TILES[_<K>] = 0/1. Tiles are handed out
// in raster order from a global counter instead of the static round robin, so the tiles in
// flight stay a contiguous stretch of the raster without the soft k-barrier (which it
// replaces for that GEMM). Default on for K1 (FWD) and K4 (DZ): K = H is short, so a raster
// group's operands stay in L2 wherever each pair is inside its tile; K4 88.6 -> 93.8%
// tensor-active with DRAM reads 7.0 -> 5.4 GB, K1 reads 7.4 -> 5.3 GB, step -0.7 ms
// (profiles/r02/dyn/, dyn2/); on for the Newton-Schulz GEMMs (split-K Gram, X C): 5 steps
// 38.7-40.0 -> 37.5-38.3 ms (profiles/r02/ns_dyn/). Off for K5 / K6, whose long K needs the
// k-lockstep of the barrier (dynamic: DRAM reads 14.7 -> 22.8 / 13.3 -> 18.2 GB). Not for the
// NVLS-fused or grouped GEMMs.
bool dyn_tiles_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_DYN_TILES", -1);
  if (kid < 0 || kid >= kKnobKids) return false;
  if (env[kid] >= 0) return env[kid] > 0;
  return kid == RL_K_FWD_GEMM || kid == RL_K_DZ_GEMM || kid == RL_K_NS_GEMM;
}
int skew() {
  static const int v = [] {
    const char* e = getenv("RL_SKEW");
    const int x = e ? atoi(e) : 3;
    return (x == 0 || x == 2) ? x : 3;
  }();
  return v;
}
// Epilogue warps of the LSE GEMM (K1): RL_EPI_WARPS[_FWD] = 4, 8 or 16 (default 8, two
// warps per TMEM lane quarter; see rl_gemm.cuh).
int epi_warps_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_EPI_WARPS", -1);
  if (kid < 0 || kid >= kKnobKids) return 4;
  return env[kid] == 4 ? 4 : (env[kid] == 16 ? 16 : 8);
}
// Epilogue warps of K6 (dW, fp32 store / reduce-add): RL_EPI_WARPS_DW = 8 (default: each warp
// loads its 4 chunks of a TMEM half at once and releases it before storing; K6 17.61 -> 17.42 M
// cycles, profiles/r02/k6_w8_early/) or 4. The NVLS-fused dW GEMM keeps 4.
int epi_warps_dw() {
  static const int v = [] {
    const char* e = getenv("RL_EPI_WARPS_DW");
    return (e && atoi(e) == 4) ? 4 : 8;
  }();
  return v;
}
int sync_slack_for(int kid) {
  static const std::array<int, kKnobKids> env = env_table("RL_SYNC_SLACK", -1);
  if (kid < 0 || kid >= kKnobKids) return 2;
  return env[kid] >= 0 ? env[kid] : 2;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: one bit per
// device and kernel instantiation records that it was set.
template <typename K>
rl_status ensure_smem_attr(K kern, int smem, std::atomic<uint64_t>& done) {
  int dev = 0;
  RL_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return RL_OK;
  RL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  done.fetch_or(bit, std::memory_order_release);
  return RL_OK;
}

constexpr int kMaxSyncPoints = 1 << 16;
thread_local uint32_t* g_sync_ctr = nullptr;  // set per call from the workspace

template <int CG, int NB>
constexpr int stages_for() {
  return CG == 2 ? (NB == 2 ? 4 : 6) : 4;
}

template <int MODE, bool A_MN, bool B_MN, int CG, int NB = 1, int SKEW = 0, int EW = 4>
rl_status launch_gemm_cg(int kid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t M,
                         int64_t N, int64_t K, int group_m, const rl::EpiParams& ep, int sms, cudaStream_t st,
                         int k_splits = 1, int split_rows = 0, const int* dyn_count = nullptr, int dyn_mode = 0) {
  constexpr int S = stages_for<CG, NB>();
  auto kern = rl::gemm_kernel<MODE, A_MN, B_MN, CG, S, NB, SKEW, EW>;
  constexpr int smem = rl::gemm_smem_bytes<CG, S, false, NB>();
  static_assert(smem <= 232448, "dynamic shared memory over 227 KB");
  static std::atomic<uint64_t> attr_done{0};  // per instantiation, one bit per device
  RL_TRY(ensure_smem_attr(kern, smem, attr_done));
  using TL = rl::Tiling<CG>;
  rl::GemmShape sh;
  sh.m_blocks = static_cast<int>((M + TL::TILE_M - 1) / TL::TILE_M);
  sh.n_blocks = static_cast<int>((N + rl::BN * NB - 1) / (rl::BN * NB));
  sh.k_blocks = static_cast<int>((K + rl::BK - 1) / rl::BK);
  sh.group_m = group_m;
  // K = 0 only for the NVLS epilogue (a rank with no rows still stores zeros, or adds
  // nothing, and takes part in the reduction of every slab)
  if (sh.k_blocks == 0 && MODE != rl::EPI_F32_NVLS) return fail(RL_ERR_SHAPE, "GEMM with K = 0");
  if (k_splits < 1 || sh.k_blocks == 0) k_splits = 1;
  if (k_splits > sh.k_blocks && sh.k_blocks > 0) k_splits = sh.k_blocks;
  sh.k_per_split = sh.k_blocks > 0 ? (sh.k_blocks + k_splits - 1) / k_splits : 0;
  sh.k_splits = sh.k_blocks > 0 ? (sh.k_blocks + sh.k_per_split - 1) / sh.k_per_split : 1;
  sh.split_rows = split_rows;
  sh.dyn_count = dyn_count;
  sh.dyn_mode = dyn_count ? dyn_mode : 0;
  if (sh.k_splits > 1 && (MODE == rl::EPI_LSE || MODE == rl::EPI_DZ || MODE == rl::EPI_F32_NVLS))
    return fail(RL_ERR_UNSUPPORTED, "split-K needs a plain store epilogue");
  const int64_t tiles = static_cast<int64_t>(sh.m_blocks) * sh.n_blocks * sh.k_splits;
  const int units = static_cast<int>(tiles < sms / CG ? tiles : sms / CG);
  rl::EpiParams ep2 = ep;
  ep2.k_serpentine = serpentine_for(kid) ? 1 : 0;
  ep2.sync_every = 0;
  ep2.dyn_tiles = 0;
  ep2.tile_ctr = nullptr;
  if (g_sync_ctr && dyn_tiles_for(kid) &&
      (MODE == rl::EPI_LSE || MODE == rl::EPI_DZ || MODE == rl::EPI_BF16 || MODE == rl::EPI_F32 ||
       MODE == rl::EPI_F32_ADD)) {
    RL_CUDA(cudaMemsetAsync(g_sync_ctr, 0, 4, st));
    ep2.dyn_tiles = 1;
    ep2.tile_ctr = reinterpret_cast<int*>(g_sync_ctr);
  } else if (g_sync_ctr && sync_every_for(kid) > 0) {
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
  cfg.blockDim = dim3(rl::kernel_threads(MODE, EW));
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

template <int MODE, bool A_MN, bool B_MN, int EW>
rl_status launch_gemm_ew(int kid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t M,
                         int64_t N, int64_t K, int group_m, const rl::EpiParams& ep, int sms, cudaStream_t st,
                         int k_splits, int split_rows, const int* dyn_count, int dyn_mode) {
  // wide tiles only where a tile covers at least two 256-column blocks
  if (cta_group() == 2 && wide_for(kid) && N > rl::BN) {
    switch (skew()) {
      case 0:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 0, EW>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                             split_rows, dyn_count, dyn_mode);
      case 2:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 2, EW>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                             split_rows, dyn_count, dyn_mode);
      default:
        return launch_gemm_cg<MODE, A_MN, B_MN, 2, 2, 3, EW>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                             split_rows, dyn_count, dyn_mode);
    }
  }
  if (cta_group() == 2)
    return launch_gemm_cg<MODE, A_MN, B_MN, 2, 1, 0, EW>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                         split_rows, dyn_count, dyn_mode);
  return launch_gemm_cg<MODE, A_MN, B_MN, 1, 1, 0, EW>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits,
                                                       split_rows, dyn_count, dyn_mode);
}

template <int MODE, bool A_MN, bool B_MN>
rl_status launch_gemm(int kid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int64_t M, int64_t N,
                      int64_t K, int group_m, const rl::EpiParams& ep, int sms, cudaStream_t st, int k_splits = 1,
                      int split_rows = 0, const int* dyn_count = nullptr, int dyn_mode = 0) {
  if (M <= 0 || N <= 0) return RL_OK;
  if constexpr (MODE == rl::EPI_F32 || MODE == rl::EPI_F32_ADD) {
    // the wide dW GEMM (K6) with 8 epilogue warps that release each TMEM half before storing
    if (kid == RL_K_DW_GEMM && epi_warps_dw() == 8 && cta_group() == 2 && wide_for(kid) && N > rl::BN)
      return launch_gemm_ew<MODE, A_MN, B_MN, 8>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
                                                 dyn_count, dyn_mode);
  }
  if constexpr (MODE == rl::EPI_LSE) {
    if (epi_warps_for(kid) == 8)
      return launch_gemm_ew<MODE, A_MN, B_MN, 8>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
                                                 dyn_count, dyn_mode);
    if (epi_warps_for(kid) == 16)
      return launch_gemm_ew<MODE, A_MN, B_MN, 16>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
                                                  dyn_count, dyn_mode);
  }
  return launch_gemm_ew<MODE, A_MN, B_MN, 4>(kid, a, b, c, M, N, K, group_m, ep, sms, st, k_splits, split_rows,
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
  static std::atomic<uint64_t> attr_done{0};
  RL_TRY(ensure_smem_attr(kern, smem, attr_done));
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

}  // namespace
