// Persistent warp-specialised tcgen05 GEMM with the path's fused epilogues.
//
//   D[m, n] = sum_k A[m, k] * B[n, k]      (bf16 in, fp32 accumulate in TMEM)
//
// CG = 1: one CTA per SM computes 128 x 256 tiles.
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes 256 x 256 tiles with
//         tcgen05.mma.cta_group::2: each CTA stages half of A (128 rows) and half
//         of B (128 rows) per k-block and holds 128 rows x 256 fp32 columns of D in
//         its own TMEM; the leader CTA issues the MMAs. Per SM this moves 2/3 of
//         the operand bytes of CG = 1 for the same FLOPs.
// BK = 64 (one 128-byte swizzle atom of bf16), a STAGES-deep TMA ring, two TMEM
// accumulators (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of
// tile i+1.
// NB = 2 (wide tiles, CG = 2): the pair computes 256 x 512 with two N = 256 MMAs
//         per k-step that share the A stage, so each SM moves 48 instead of 64 bytes
//         from L2 per 1024 MMA cycles (3/4). The one accumulator then fills all 512
//         TMEM columns; the first / last SKEW k-blocks of a tile run block 0 before
//         block 1, so each TMEM half drains under the other half's MMAs (K1, K5, K6).
// Warp roles: warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer (leader
// CTA), warps 2 .. 2+EW-1 = epilogue (thread = accumulator row; EW = 8 for K1:
// two warps per TMEM lane quarter), and for EPI_F32_NVLS 4 more communication
// warps that run the cross-rank slab reductions (comm_warps()).
// Order of k-blocks: ascending, or serpentine (tiles of odd waves backwards,
// EpiParams::k_serpentine) for K6 / Newton-Schulz. Tile order: static round robin
// (tile = pair + i * pairs) with a soft k-barrier between the producers that keeps the
// CTAs sharing operands inside one L2 window (sync_*), or dynamic (dyn_tiles): each
// pair's leader producer takes the next tile of the raster from a global counter and
// passes it to every role of both CTAs through a shared-memory ring (next_tile).
//
// Epilogues:
//   EPI_LSE  (K1): per row of the tile, online (m, s, u, z_target) over the
//                  tile's 256 scaled logits -> one float4 partial per (n-tile, row).
//                  Logits never leave TMEM/registers.
//   EPI_DZ   (K4): dU = coef*invT*(exp(z - lse) - [v == y]) -> bf16 -> TMA store.
//   EPI_BF16 (K5): plain bf16 store.   EPI_F32 / EPI_F32_ADD (K5/K6): fp32 store
//                  or TMA reduce-add into the destination.
//   EPI_F32_NVLS (K5/K6 multi-GPU): fp32 store into this rank's replica of a
//                  symmetric buffer + the NVLink-multicast reduction.
//   EPI_BF16_GROUPED (MoE): masked bf16 stores per expert group, optional row scale.
#pragma once
#include "rl_ptx.cuh"

namespace rl {

constexpr int BN = 256, BK = 64;
constexpr int gemm_threads(int epi_warps) { return 64 + 32 * epi_warps; }
constexpr int GEMM_THREADS = gemm_threads(4);  // the 4-epilogue-warp kernels (grouped GEMM, diagnostics)
// EPI_F32_NVLS adds 4 communication warps (one per TMEM lane quarter's slabs) that run the
// cross-rank reductions, so the epilogue warps only drain TMEM, store and publish
constexpr int comm_warps(int mode);
constexpr int kernel_threads(int mode, int epi_warps) { return gemm_threads(epi_warps) + 32 * comm_warps(mode); }
constexpr int EPI_BUF_BYTES = 32 * 128;  // one warp's 32-row x 128-byte store chunk
constexpr int EPI_BYTES = 4 * 2 * EPI_BUF_BYTES;
constexpr int BAR_BYTES = 256;

enum EpiMode {
  EPI_LSE = 0,
  EPI_DZ = 1,
  EPI_BF16 = 2,
  EPI_F32 = 3,
  EPI_F32_ADD = 4,
  EPI_F32_NVLS = 5,
  EPI_BF16_GROUPED = 6  // grouped GEMM (MoE experts): row groups from device offsets, masked bf16 stores
};
constexpr int MAX_GROUPS = 1024;
constexpr int comm_warps(int mode) { return mode == EPI_F32_NVLS ? 4 : 0; }

constexpr int NVLS_MAX_RANKS = 8;

#ifdef RL_AB_K4_NOSTORE
__device__ unsigned g_ab_k4_launches = 0;  // A/B build only: K4 launches so far
#endif
#ifdef RL_AB_STATS
// A/B build only: per-CTA cycle counters of the last launch of each epilogue mode
// [mode][cta][slot]: 0 MMA waits on tempty, 1 MMA waits on full, 2 MMA loop total,
// 3 producer waits on empty, 4 producer k-barrier waits, 5 epilogue (warp 2) waits on
// tfull, 6 epilogue (warp 2) drain cycles, 7 tiles
__device__ unsigned long long g_ab_stats[8][512][8];
#define RL_AB_CLK(v) const long long v = clock64()
// accumulate in registers (ab_acc[], per thread); RL_AB_FLUSH writes them out once
#define RL_AB_ADD(slot, t0) ab_acc[slot] += static_cast<unsigned long long>(clock64() - (t0))
#define RL_AB_FLUSH(slot) g_ab_stats[MODE][blockIdx.x][slot] = ab_acc[slot]
#else
#define RL_AB_FLUSH(slot)
#define RL_AB_CLK(v)
#define RL_AB_ADD(slot, t0)
#endif

template <int CG>
struct Tiling {
  static constexpr int TILE_M = 128 * CG;          // output rows per tile (per CTA pair)
  static constexpr int A_ROWS = 128;               // A rows staged per CTA
  static constexpr int B_ROWS = BN / CG;           // B rows (n) staged per CTA
  static constexpr int A_STAGE = A_ROWS * BK * 2;  // bytes per stage per CTA
  static constexpr int B_STAGE = B_ROWS * BK * 2;
  static constexpr int STAGE = A_STAGE + B_STAGE;
};

template <int CG, int STAGES, bool GROUPED = false, int NB = 1>
constexpr int gemm_smem_bytes() {
  return 1024 + STAGES * (Tiling<CG>::A_STAGE + NB * Tiling<CG>::B_STAGE) + EPI_BYTES + BAR_BYTES +
         (GROUPED ? (MAX_GROUPS + 1) * 4 : 0);
}

struct GemmShape {
  int m_blocks, n_blocks, k_blocks;  // m_blocks counts TILE_M-row tiles
  int group_m;                       // raster: tiles walk n inside groups of group_m m-blocks
  int k_splits;                      // split-K: tile t covers k-blocks of split t / (m_blocks*n_blocks)
  int k_per_split;                   // k-blocks per split
  int split_rows;                    // store epilogues: split s writes rows offset by s*split_rows
  // device-side problem size (sparse backward): dyn_mode 1 = M rows, 2 = K rows come
  // from *dyn_count at kernel start (the host sized the grid for the upper bound)
  const int* dyn_count;
  int dyn_mode;
};

__device__ __forceinline__ void tile_k_range(int tile, const GemmShape& sh, int& kb0, int& kb1) {
  const int ks = tile / (sh.m_blocks * sh.n_blocks);
  kb0 = ks * sh.k_per_split;
  kb1 = min(sh.k_blocks, kb0 + sh.k_per_split);
}

struct EpiParams {
  int64_t rows;          // valid rows of D (M)
  int64_t cols;          // valid columns of D (N)
  float scale_log2;      // invT * log2(e)
  float inv_temperature; // invT
  // EPI_LSE / EPI_DZ
  const int32_t* targets;  // [rows] global ids, row-indexed from D's row 0
  int64_t vocab_offset;    // global id of D's column 0
  float4* partials;        // EPI_LSE: [n_blocks][rows]
  const float* lse;        // EPI_DZ:  [rows]
  const float* coef;       // EPI_DZ:  [rows]
  const float* invt_rows;  // EPI_LSE / EPI_DZ: optional per-row 1/tau (R20), else inv_temperature
  // soft k-barrier (locality): producers of all CTAs arrive on sync_ctr[p] every
  // sync_every k-blocks and do not run more than sync_slack points ahead of the
  // slowest CTA, so CTAs sharing operands stay inside one L2 window. 0 = off.
  uint32_t* sync_ctr;      // [max_sync + 1], zeroed before the launch
  int sync_every;
  int sync_slack;
  int max_sync;            // highest sync point any CTA reaches
  int k_serpentine;        // odd tiles of a CTA walk their k-blocks backwards (L2 reuse across waves)
  // EPI_F32_NVLS: D is also reduced over the ranks of an NVLink multicast group.
  // Every warp stores its 32-row slab locally (TMA), then publishes flag[slab] =
  // epoch; the rank owning the tile (tile % world) later sums the slab over all
  // replicas with multimem.ld_reduce and writes the sum to all with multimem.st.
  // EPI_BF16_GROUPED: D rows [off[g], off[g+1]) = A rows of the group times B_g^T,
  // B_g = rows [g * cols, (g + 1) * cols) of B; D is bf16 [rows][cols] at `grouped_out`.
  const int32_t* group_offsets;            // [n_groups + 1], device
  int n_groups;
  uint16_t* grouped_out;
  const float* row_scale;                  // optional [rows]: D[r, :] *= row_scale[r] (fused RMSNorm)
  float* nvls_mc;                          // multicast VA of D ([rows][cols], fp32)
  uint32_t* nvls_flags[NVLS_MAX_RANKS];    // every rank's flag array ([rank] is local)
  int nvls_rank, nvls_world;
  uint32_t nvls_epoch;
  int nvls_lag;                            // 0: the communication warps reduce each slab once every
                                           // rank published it; > 0: the epilogue warps reduce the
                                           // slab finished this many tiles ago (round-1 schedule)
  int nvls_mode;                           // 0 all-reduce (owner tile % world), 1 reduce-scatter by rows
  int64_t nvls_shard;                      // mode 1: rows per rank (a multiple of 32)
  float* nvls_local;                       // mode 1 / row_map: this rank's replica (plain stores)
  int nvls_add;                            // the local store adds to D (TMA reduce-add): D already
                                           // holds earlier chunks / micro-batches of this rank
  // EPI_F32_NVLS with a row map (sparse backward, compacted rows): D row r is output
  // row row_map[r] of nvls_local / nvls_mc (rows >= the device row count are skipped);
  // the store is a plain per-row global store instead of TMA
  const int32_t* row_map;
  int* tile_ctr;
  int dyn_tiles;
  // EPI_LSE probability cache (K4 from the cache instead of the recompute GEMM): for every
  // 32-column chunk, p_out[(p_row0 + row) * p_ld + col] = fp16(2^(z sl2 - m)) with m the row's
  // running max after the chunk (log2 units, >= every value of the chunk), and
  // p_m[(col / 32) * p_rows + p_row0 + row] = m. nullptr = off.
  uint16_t* p_out;
  float* p_m;
  int64_t p_ld, p_row0, p_rows;
  int p_evict_first;  // direct stores of the cache with an L2 evict-first policy
  int p_tma;          // tmC maps the cache (32 x 32 boxes, 64B swizzle): 8-warp epilogues stage each
                      // chunk in shared memory and TMA-store it
};

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tile_coords(int tile, const GemmShape& sh, int& m, int& n) {
  tile %= sh.m_blocks * sh.n_blocks;  // split-K: the split index is the outer coordinate
  const int per_group = sh.group_m * sh.n_blocks;
  const int g = tile / per_group;
  const int first_m = g * sh.group_m;
  const int gsize = min(sh.group_m, sh.m_blocks - first_m);
  const int r = tile - g * per_group;
  m = first_m + r % gsize;
  n = r / gsize;
}

// Write one thread's 128-byte row chunk into a 128B-swizzled 32-row staging buffer.
__device__ __forceinline__ void stage_row(uint32_t buf, int row, const uint32_t (&w)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t addr = buf + row * 128 + ((j ^ (row & 7)) << 4);
    st_shared_v4(addr, w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }
}

// Group row range, clamped to [0, rows] and to a non-decreasing sequence, so bad
// offsets can skip work but never address memory outside A or D.
__device__ __forceinline__ int grp_begin(const EpiParams& ep, int g) {
  const int64_t v = ep.group_offsets[g];
  return static_cast<int>(v < 0 ? 0 : (v > ep.rows ? ep.rows : v));
}
__device__ __forceinline__ int grp_end(const EpiParams& ep, int g) {
  const int64_t v = ep.group_offsets[g + 1];
  const int e = static_cast<int>(v < 0 ? 0 : (v > ep.rows ? ep.rows : v));
  const int b = grp_begin(ep, g);
  return e < b ? b : e;
}

// Slab = 32 accumulator rows of one tile owned by one epilogue warp.
__device__ __forceinline__ int nvls_slab(int tile, uint32_t rank, int q) { return tile * 8 + rank * 4 + q; }

// Owner-side reduction of one slab over the multicast group (see EpiParams::nvls_*).
// Flags hold the epoch of the last call that published the slab; epochs increase
// from call to call (and chunk to chunk), so a rank that already moved on to a later
// chunk still satisfies the wait (its later chunk writes other rows).
template <int TILE_M, int TN>
__device__ __noinline__ void nvls_reduce_slab_impl(const EpiParams& ep, const GemmShape& sh, int tile, uint32_t rank,
                                                   int q, int lane, int64_t rows_valid) {
  int m, n;
  tile_coords(tile, sh, m, n);
  const int64_t r0 = static_cast<int64_t>(m) * TILE_M + rank * 128 + q * 32;
  if (ep.nvls_mode == 0) {
    if (tile % ep.nvls_world != ep.nvls_rank) return;
  } else {
    const int64_t own = r0 / ep.nvls_shard;
    if ((own < ep.nvls_world ? own : ep.nvls_world - 1) != ep.nvls_rank || r0 >= ep.rows) return;
  }
  const int slab = nvls_slab(tile, rank, q);
  if (lane < ep.nvls_world) {
    const uint32_t* f = ep.nvls_flags[lane] + slab;
    const long long t0 = clock64();
    while (ld_acquire_sys(f) < ep.nvls_epoch) {
      __nanosleep(128);
      if (clock64() - t0 > (1ll << 36)) __trap();
    }
  }
  __syncwarp();
  const int64_t c0 = static_cast<int64_t>(n) * TN;
  const int64_t rleft = rows_valid - r0, cleft = ep.cols - c0;
  if (rleft <= 0) return;
  const int rmax = rleft < 32 ? static_cast<int>(rleft) : 32;
  const int cmax = cleft < TN ? static_cast<int>(cleft) : TN;
  // output row of slab row i (compacted rows are scattered through the row map)
  auto orow = [&](int i) -> int64_t { return ep.row_map ? static_cast<int64_t>(ep.row_map[r0 + i]) : r0 + i; };
  // lane l covers columns 4l..4l+3, 128+4l.., ...: TN/128 x 16 B per row, 16 loads in flight
  constexpr int H = TN / 128, RB = 16 / H;
  for (int rb = 0; rb < rmax; rb += RB) {
    float v[RB][H][4];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int c = h * 128 + lane * 4;
        if (rb + i < rmax && c < cmax) mc_ld_reduce_v4(ep.nvls_mc + orow(rb + i) * ep.cols + c0 + c, v[i][h]);
      }
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int c = h * 128 + lane * 4;
        if (rb + i < rmax && c < cmax) {
          const int64_t off = orow(rb + i) * ep.cols + c0 + c;
          if (ep.nvls_mode == 0)
            mc_st_v4(ep.nvls_mc + off, v[i][h]);
          else
            *reinterpret_cast<float4*>(ep.nvls_local + off) = make_float4(v[i][h][0], v[i][h][1], v[i][h][2], v[i][h][3]);
        }
      }
  }
}

// EW = epilogue warps: 4 (one per TMEM lane quarter), or 8 for EPI_LSE (two per lane
// quarter, each taking half of a TMEM half's 256 columns; the pair merges its online
// softmax states through shared memory): the drain of a TMEM half is bound by TMEM reads
// (64 B/clk per SM) and the exponentials, and a second warp per SM sub-partition keeps a
// load in flight while the other computes.
template <int MODE, bool A_MN, bool B_MN, int CG, int STAGES, int NB = 1, int SKEW = 0, int EW = 4>
__global__ void __launch_bounds__(kernel_threads(MODE, EW), 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const GemmShape sh_in, const EpiParams ep) {
  using TL = Tiling<CG>;
  static_assert(NB == 1 || (NB == 2 && CG == 2 && MODE != EPI_BF16_GROUPED), "wide tiles: CTA pairs, not grouped");
  static_assert(SKEW < STAGES, "the skewed head/tail holds SKEW stages");
  static_assert(EW == 4 || ((EW == 8 || EW == 16) && MODE == EPI_LSE) ||
                    (EW == 8 && (MODE == EPI_DZ || MODE == EPI_F32 || MODE == EPI_F32_ADD)),
                "more epilogue warps: LSE (8 / 16), dU and fp32 store (8) epilogues only");
  constexpr int TN = BN * NB;                 // tile columns
  constexpr int kStoreGroups = NB * (BN / 32);  // fp32 store epilogues: bulk groups per tile and warp
  constexpr int NACC = NB == 1 ? 2 : 1;       // TMEM accumulators (512 columns in total)
  constexpr int B_STAGE_ALL = NB * TL::B_STAGE;
  GemmShape sh = sh_in;
  int64_t rows_valid = ep.rows;  // D rows that hold data (dyn_mode 1: the device row count)
  if (sh.dyn_mode != 0) {
    const int cnt = *sh.dyn_count;
    if (sh.dyn_mode == 1) {
      sh.m_blocks = (cnt + TL::TILE_M - 1) / TL::TILE_M;
      if (cnt < rows_valid) rows_valid = cnt;
    } else {
      sh.k_blocks = (cnt + BK - 1) / BK;
      sh.k_per_split = sh.k_blocks;
      sh.k_splits = 1;
    }
  }
#ifdef RL_AB_STATS
  unsigned long long ab_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
#ifdef RL_AB_K4_NOSTORE
  const bool ab_k4_skip = MODE == EPI_DZ && *(volatile unsigned*)&g_ab_k4_launches > 0;
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * TL::A_STAGE;
  uint8_t* sEpi = sB + STAGES * B_STAGE_ALL;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // dynamic tile ring (EpiParams::dyn_tiles): TR slots after the TMEM slot
  constexpr bool kDynOk = MODE == EPI_LSE || MODE == EPI_DZ || MODE == EPI_BF16 || MODE == EPI_F32 || MODE == EPI_F32_ADD;
  constexpr int TR = 4;
  static_assert(2 * STAGES + 4 <= 16 && (17 + 2 * TR) * 8 + TR * 4 <= BAR_BYTES, "barrier area");
  uint64_t* rfull = full + 17;
  uint64_t* rempty = rfull + TR;
  int* rslot = reinterpret_cast<int*>(rempty + TR);
  constexpr bool GROUPED = MODE == EPI_BF16_GROUPED;
  int* s_prefix = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full) + BAR_BYTES);  // GROUPED only

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG;  // CTA pair (or CTA) index
  const int n_units = gridDim.x / CG;

  if (threadIdx.x == 0) {
#ifdef RL_AB_STATS
    for (int k = 0; k < 8; ++k) g_ab_stats[MODE][blockIdx.x][k] = 0;
#endif
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EW * CG);
    }
    if constexpr (kDynOk) {
      for (int r = 0; r < TR; ++r) {
        mbar_init(&rfull[r], 1);
        mbar_init(&rempty[r], CG == 2 ? 2 + 2 * EW : 1 + EW);
      }
    }
    fence_mbar_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (MODE != EPI_LSE) tma_prefetch(&tmC);
  }
  if constexpr (GROUPED) {
    // tiles per group: ceil(rows_g / TILE_M) * n_blocks (n fastest inside a group); the
    // counts are loaded by all threads in parallel, then prefix-summed from smem
    for (int g = threadIdx.x; g < ep.n_groups; g += blockDim.x) {
      const int rows_g = grp_end(ep, g) - grp_begin(ep, g);
      s_prefix[g + 1] = (rows_g + TL::TILE_M - 1) / TL::TILE_M * sh.n_blocks;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_prefix[0] = 0;
      for (int g = 1; g <= ep.n_groups; ++g) s_prefix[g] += s_prefix[g - 1];
    }
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      tmem_alloc2(tmem_slot, 512);
      tmem_relinquish2();
    } else {
      tmem_alloc(tmem_slot, 512);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = GROUPED ? s_prefix[ep.n_groups] : sh.m_blocks * sh.n_blocks * sh.k_splits;
  // grouped tiles -> (group, first A row, row end, n); otherwise the raster of tile_coords
  auto group_tile = [&](int tile, int& g, int& row0, int& row_end, int& n) {
    int lo = 0, hi = ep.n_groups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    g = lo;
    const int local = tile - s_prefix[g];
    row0 = grp_begin(ep, g) + (local / sh.n_blocks) * TL::TILE_M;
    row_end = grp_end(ep, g);
    n = local % sh.n_blocks;
  };

  // Tile ti of this CTA's sequence (-1: none left; prev = tile ti - 1), called by whole warps
  // in order. Static: unit + ti * n_units. Dynamic: the pair leader's producer takes tiles from the global
  // counter and writes each into slot ti % TR of both CTAs' rings; every other role reads
  // its slot and releases it on the leader's ring barrier. Either way a tile's k-blocks run
  // on one pair in a fixed order, so the results do not depend on the schedule.
  const bool dyn = kDynOk && ep.dyn_tiles != 0;
  int* const tile_ctr = ep.tile_ctr;
  // (captures by value: a by-reference capture costs K1 stack space)
  auto next_tile = [=](int ti, int prev) -> int {
    if (!kDynOk || !dyn) {
      const int t = prev + n_units;
      return t < total ? t : -1;
    }
    const int r = ti & (TR - 1);
    const uint32_t par = static_cast<uint32_t>(ti / TR) & 1u;
    if (warp == 0 && leader) {
      mbar_wait_cluster(&rempty[r], par ^ 1u);
      int t = 0;
      if (lane == 0) {
        t = atomicAdd(tile_ctr, 1);
        if (t >= total) t = -1;
        rslot[r] = t;
        if constexpr (CG == 2) {
          st_shared_cluster_s32(mapa_shared(smem_u32(&rslot[r]), 1), t);
          mbar_arrive_cluster(mapa_shared(smem_u32(&rfull[r]), 1));
        }
        mbar_arrive(&rfull[r]);
      }
      return __shfl_sync(0xffffffffu, t, 0);
    }
    mbar_wait_cluster(&rfull[r], par);
    const int t = *reinterpret_cast<volatile int*>(&rslot[r]);
    __syncwarp();
    if (lane == 0) {
      if constexpr (CG == 2)
        mbar_arrive_cluster(mapa_shared(smem_u32(&rempty[r]), 0));
      else
        mbar_arrive(&rempty[r]);
    }
    return t;
  };

  if (warp == 0) {
    // ------------------------------------------------------------- producer
    // The whole warp walks the schedule (warp-uniform state lives in uniform
    // registers); one elected lane issues the TMA copies.
    int s = 0;
    uint32_t ph = 0;
    int gk = 0;            // k-blocks issued by this CTA so far (all tiles)
    int last_sync = 0;
    for (int ti = 0, tile = next_tile(0, unit - n_units); tile >= 0; ++ti, tile = next_tile(ti, tile)) {
      int m, n, a_row, b_row;
      if constexpr (GROUPED) {
        int g, row0, row_end;
        group_tile(tile, g, row0, row_end, n);
        a_row = row0 + rank * TL::A_ROWS;
        b_row = static_cast<int>(g * ep.cols) + n * BN + rank * TL::B_ROWS;
        (void)m;
      } else {
        tile_coords(tile, sh, m, n);
        a_row = m * TL::TILE_M + rank * TL::A_ROWS;
        b_row = n * TN + rank * TL::B_ROWS;
      }
      int kb0 = 0, kb1 = sh.k_blocks;
      if constexpr (!GROUPED) tile_k_range(tile, sh, kb0, kb1);
      // serpentine: the MMA accumulates in issue order, so only the loads are reordered
      const bool k_rev = ep.k_serpentine && ((tile / n_units) & 1);
      for (int kb_i = kb0; kb_i < kb1; ++kb_i, ++gk) {
        const int kb = k_rev ? kb0 + kb1 - 1 - kb_i : kb_i;
        if (ep.sync_every > 0 && gk > 0 && gk % ep.sync_every == 0) {
          const int p = gk / ep.sync_every;
          if (lane == 0) {
            red_release_add(ep.sync_ctr + p, 1u);
            if (p > ep.sync_slack) {
              // a locality hint, never a dependency: give up after ~2^17 cycles so a
              // CTA that cannot become resident (shared GPU) cannot stall the others
              const uint32_t* c = ep.sync_ctr + (p - ep.sync_slack);
              const long long t0 = clock64();
              while (ld_acquire(c) < gridDim.x && clock64() - t0 < (1ll << 17)) __nanosleep(64);
              RL_AB_ADD(4, t0);
            }
          }
          __syncwarp();
          last_sync = p;
        }
        {
          RL_AB_CLK(tw);
          mbar_wait_sleep(&empty[s], ph ^ 1);
          if (lane == 0) RL_AB_ADD(3, tw);
        }
        if (elect_one()) {
          if (leader) mbar_expect_tx(&full[s], CG * (TL::A_STAGE + B_STAGE_ALL));
          int k0 = kb * BK;
#ifdef RL_AB_DU_L2
          // A/B measurement only (never in the product build): K5 / K6 read their dU
          // operand from a 256-row window (77 MB at V = 151552) that stays in L2, i.e. a
          // backward whose dU never reaches DRAM; the outputs are garbage
          if (MODE == EPI_BF16 && !A_MN && B_MN) a_row &= 255;
          if (MODE == EPI_F32 && A_MN && B_MN) k0 &= 255;
#endif
          uint8_t* a = sA + s * TL::A_STAGE;
          uint8_t* b = sB + s * B_STAGE_ALL;
          if constexpr (CG == 2) {
            if (!A_MN) {
              tma_load_2d_pair(a, &tmA, &full[s], k0, a_row);
            } else {
              tma_load_2d_pair(a, &tmA, &full[s], a_row, k0);
              tma_load_2d_pair(a + 8192, &tmA, &full[s], a_row + 64, k0);
            }
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              // block nb: columns nb*256.. of the tile; this CTA holds its half (128)
              uint8_t* bb = b + nb * TL::B_STAGE;
              const int br = b_row + nb * BN;
              if (!B_MN) {
                tma_load_2d_pair(bb, &tmB, &full[s], k0, br);
              } else {
#pragma unroll
                for (int j = 0; j < TL::B_ROWS / 64; ++j)
                  tma_load_2d_pair(bb + j * 8192, &tmB, &full[s], br + 64 * j, k0);
              }
            }
          } else {
            if (!A_MN) {
              tma_load_2d(a, &tmA, &full[s], k0, a_row);
            } else {
              tma_load_2d(a, &tmA, &full[s], a_row, k0);
              tma_load_2d(a + 8192, &tmA, &full[s], a_row + 64, k0);
            }
            if (!B_MN) {
              tma_load_2d(b, &tmB, &full[s], k0, b_row);
            } else {
#pragma unroll
              for (int j = 0; j < TL::B_ROWS / 64; ++j)
                tma_load_2d(b + j * 8192, &tmB, &full[s], b_row + 64 * j, k0);
            }
          }
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    // arrive on the sync points this CTA never reaches (it had fewer tiles)
    if (ep.sync_every > 0 && lane == 0)
      for (int p = last_sync + 1; p <= ep.max_sync; ++p) red_release_add(ep.sync_ctr + p, 1u);
    if (lane == 0) {
      RL_AB_FLUSH(3);
      RL_AB_FLUSH(4);
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    if constexpr (NB == 2) {
      // Wide tiles: TMEM half h (columns h*256..) accumulates the N = 256 block h. The
      // first and last D k-blocks of a tile run block 0 before block 1, so the
      // epilogue drains half 0 of tile i while block 1 finishes its tail, and half 1
      // while block 0 of tile i+1 runs its head (D*512 MMA cycles of cover each).
      // One op per (k-block, block set), one issue site (keeps the kernel small):
      //   ops [0, D)            head, block 0      (wait full)
      //   ops [D, 2D)           head, block 1      (release stage)
      //   ops [2D, L)           both blocks        (wait full, release stage)
      //   ops [L, L+D)          tail, block 0      (wait full), then tfull[0]
      //   ops [L+D, L+2D)       tail, block 1      (release stage), then tfull[1]
      if (leader) {
        RL_AB_CLK(t_mma0);
        constexpr uint32_t idesc = umma_idesc_bf16(TL::TILE_M, BN, A_MN, B_MN);
        uint32_t aph = 0;
        int g0 = 0;  // k-blocks consumed before this tile (stage = g % STAGES)
        const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
        for (int ti = 0, tile = next_tile(0, unit - n_units); tile >= 0; ++ti, tile = next_tile(ti, tile)) {
          int kb0 = 0, kb1 = sh.k_blocks;
          tile_k_range(tile, sh, kb0, kb1);
          const int L = kb1 > kb0 ? kb1 - kb0 : 0;
          const int D = SKEW < L / 2 ? SKEW : L / 2;
          {
            RL_AB_CLK(tw);
            mbar_wait(&tempty[0], aph ^ 1);
            if (D == 0) mbar_wait(&tempty[1], aph ^ 1);
            if (lane == 0) RL_AB_ADD(0, tw);
          }
          tc_fence_after();
#pragma unroll 1
          for (int op = 0; op < L + 2 * D; ++op) {
            int j, nb_lo, nb_hi;
            bool wait_full, release;
            if (op < D) { j = op; nb_lo = 0; nb_hi = 0; wait_full = true; release = false; }
            else if (op < 2 * D) { j = op - D; nb_lo = 1; nb_hi = 1; wait_full = false; release = true; }
            else if (op < L) { j = op - D; nb_lo = 0; nb_hi = 1; wait_full = true; release = true; }
            else if (op < L + D) { j = op - D; nb_lo = 0; nb_hi = 0; wait_full = true; release = false; }
            else { j = op - 2 * D; nb_lo = 1; nb_hi = 1; wait_full = false; release = true; }
            if (op == D && D > 0) {
              RL_AB_CLK(tw);
              mbar_wait(&tempty[1], aph ^ 1);
              if (lane == 0) RL_AB_ADD(0, tw);
              tc_fence_after();
            }
            const int g = g0 + j;
            const int st = g % STAGES;
            if (wait_full) {
              RL_AB_CLK(tw);
              mbar_wait(&full[st], (g / STAGES) & 1);
              if (lane == 0) RL_AB_ADD(1, tw);
              tc_fence_after();
            }
            if (elect_one()) {
              const uint32_t a0 = a_base + st * TL::A_STAGE;
#pragma unroll 1
              for (int nb = nb_lo; nb <= nb_hi; ++nb) {
                const uint32_t bn = b_base + st * B_STAGE_ALL + nb * TL::B_STAGE;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                  const uint64_t ad =
                      A_MN ? sw128_desc(a0 + k * 2048, 8192, 1024) : sw128_desc(a0 + k * 32, 16, 1024);
                  const uint64_t bd =
                      B_MN ? sw128_desc(bn + k * 2048, 8192, 1024) : sw128_desc(bn + k * 32, 16, 1024);
                  umma_bf16_pair(tmem_base + nb * BN, ad, bd, idesc, (j != 0) || (k != 0));
                }
              }
              if (release) umma_commit_pair(&empty[st], 0x3);
              if (op == L + D - 1 || (D == 0 && op == L - 1)) umma_commit_pair(&tfull[0], 0x3);
              if (op == L + 2 * D - 1) umma_commit_pair(&tfull[1], 0x3);
            }
            __syncwarp();
          }
          if (L == 0 && elect_one()) {  // empty K range: nothing to wait for
            umma_commit_pair(&tfull[0], 0x3);
            umma_commit_pair(&tfull[1], 0x3);
          }
          __syncwarp();
          g0 += L;
          aph ^= 1;
#ifdef RL_AB_STATS
          ab_acc[7] += 1;
#endif
        }
        if (lane == 0) {
          RL_AB_ADD(2, t_mma0);
          RL_AB_FLUSH(0); RL_AB_FLUSH(1); RL_AB_FLUSH(2); RL_AB_FLUSH(7);
        }
      }
    } else if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(TL::TILE_M, BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      RL_AB_CLK(t_mma0);
      for (int ti = 0, tile = next_tile(0, unit - n_units); tile >= 0; ++ti, tile = next_tile(ti, tile)) {
        {
          RL_AB_CLK(tw);
          mbar_wait(&tempty[acc], aph ^ 1);
          if (lane == 0) RL_AB_ADD(0, tw);
        }
        tc_fence_after();
        const uint32_t d = tmem_base + acc * TN;
        int kb0 = 0, kb1 = sh.k_blocks;
        if constexpr (!GROUPED) tile_k_range(tile, sh, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            RL_AB_CLK(tw);
            mbar_wait(&full[s], ph);
            if (lane == 0) RL_AB_ADD(1, tw);
          }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = a_base + s * TL::A_STAGE;
            const uint32_t b0 = b_base + s * B_STAGE_ALL;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = A_MN ? sw128_desc(a0 + k * 2048, 8192, 1024) : sw128_desc(a0 + k * 32, 16, 1024);
#pragma unroll
              for (int nb = 0; nb < NB; ++nb) {
                const uint32_t bn = b0 + nb * TL::B_STAGE;
                const uint64_t bd =
                    B_MN ? sw128_desc(bn + k * 2048, 8192, 1024) : sw128_desc(bn + k * 32, 16, 1024);
                if constexpr (CG == 2)
                  umma_bf16_pair(d + nb * BN, ad, bd, idesc, (kb != kb0) || (k != 0));
                else
                  umma_bf16(d + nb * BN, ad, bd, idesc, (kb != kb0) || (k != 0));
              }
            }
            if constexpr (CG == 2)
              umma_commit_pair(&empty[s], 0x3);
            else
              umma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (CG == 2)
            umma_commit_pair(&tfull[acc], 0x3);
          else
            umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (NACC == 2) acc ^= 1;
        if (acc == 0) aph ^= 1;
#ifdef RL_AB_STATS
        ab_acc[7] += 1;
#endif
      }
      if (lane == 0) {
        RL_AB_ADD(2, t_mma0);
        RL_AB_FLUSH(0); RL_AB_FLUSH(1); RL_AB_FLUSH(2); RL_AB_FLUSH(7);
      }
    }
  } else if (warp >= 2 + EW) {
    // ------------------------------------------------ communication (EPI_F32_NVLS)
    // Warp 2 + EW + q owns lane quarter q's slabs: for every tile of this CTA, wait until
    // every rank published the slab, and (if this rank owns it) sum it over the replicas
    // through the switch. Nothing here touches TMEM, so the MMA never waits for it.
    if constexpr (MODE == EPI_F32_NVLS) {
      if (ep.nvls_lag == 0) {
        const int cq = (warp - 2 - EW) & 3;
        for (int tile = unit; tile < total; tile += n_units)
          nvls_reduce_slab_impl<TL::TILE_M, TN>(ep, sh, tile, rank, cq, lane, rows_valid);
        fence_sys();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int cgrp = (warp - 2) / 4;  // EW = 8: which 128 of a TMEM half's 256 columns
    const int r_in_tile = rank * 128 + q * 32 + lane;
    // store staging: two 4 KB buffers per warp with 4 epilogue warps, one with 8 (the same
    // EPI_BYTES); EW > 4 store epilogues split each TMEM half's chunks between the warps
    // of a lane quarter
    constexpr int NBUF = EW == 4 ? 2 : 1;
    const uint32_t buf0 = smem_u32(sEpi + (warp - 2) * NBUF * EPI_BUF_BYTES);
    const uint32_t tempty_leader0 = (CG == 2) ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
    int acc = 0;
    uint32_t aph = 0;
    int chunk_ctr = 0;
    int merge_ctr = 0;  // EW = 8 LSE merges done
    int it = 0;  // tile iteration of this CTA
    auto nvls_reduce_slab = [&](const EpiParams& e, const GemmShape& g, int t, uint32_t r, int qq, int l) {
      nvls_reduce_slab_impl<TL::TILE_M, TN>(e, g, t, r, qq, l, rows_valid);
    };
#ifdef RL_AB_STATS
    long long t_drain0_shared = 0;
#endif
    auto release_tmem = [&](int a) {
      tc_fence_before();
      __syncwarp();
#ifdef RL_AB_STATS
      if (warp == 2 && lane == 0) RL_AB_ADD(6, t_drain0_shared);
#endif
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(tempty_leader0 + a * 8);
        else
          mbar_arrive(&tempty[a]);
      }
    };
    for (int ti = 0, tile = next_tile(0, unit - n_units); tile >= 0; ++ti, tile = next_tile(ti, tile)) {
      int m = 0, n;
      int64_t row;
      bool row_ok;
      int tile_row0 = 0;        // first D row of the tile (grouped)
      bool masked = false;      // grouped tile crossing a group end or the N tail
      if constexpr (GROUPED) {
        int g, row0, row_end;
        group_tile(tile, g, row0, row_end, n);
        row = static_cast<int64_t>(row0) + r_in_tile;
        row_ok = row < row_end;
        tile_row0 = row0;
        masked = row0 + TL::TILE_M > row_end || static_cast<int64_t>(n + 1) * BN > ep.cols;
      } else {
        tile_coords(tile, sh, m, n);
        row = static_cast<int64_t>(m) * TL::TILE_M + r_in_tile;
        row_ok = row < ep.rows;
      }
      // K1, 8 epilogue warps, wide tiles: one register set carries half 1 from the h = 0 pass
      // into the h = 1 pass (see the EPI_LSE branch)
      [[maybe_unused]] uint32_t lse_pre[(MODE == EPI_LSE && EW == 8 && NB == 2) ? 4 : 1][32];
#pragma unroll 1
      for (int h = 0; h < NB; ++h) {
        const int bi = NB == 2 ? h : acc;  // TMEM half (wide tiles) or accumulator
        const int n0 = n * TN + h * BN;
        {
          RL_AB_CLK(tw);
          mbar_wait_sleep(&tfull[bi], aph);
          if (warp == 2 && lane == 0) RL_AB_ADD(5, tw);
        }
#ifdef RL_AB_STATS
        t_drain0_shared = clock64();
#endif
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + bi * BN;

#ifdef RL_AB_K1_NOEPI
        // A/B measurement only: K1's epilogue releases the TMEM half without reading it
        // (no partials are written): separates the MMA loop from the drain
        if constexpr (MODE == EPI_LSE) {
          release_tmem(bi);
          continue;
        }
#endif
        if constexpr (MODE == EPI_LSE) {
          int64_t y = row_ok ? static_cast<int64_t>(ep.targets[row]) - ep.vocab_offset : -1;
          if (y >= ep.cols) y = -1;  // target lives in another vocab shard
          const int64_t tl64 = y - n0;
          const int tl = (tl64 >= 0 && tl64 < BN) ? static_cast<int>(tl64) : -1;
          const int64_t nv64 = ep.cols - n0;
          const int nvalid = nv64 < BN ? static_cast<int>(nv64) : BN;
          float mrun = -1e30f, srun = 0.f, trun = 0.f, zt = -INFINITY;
          const float it = (ep.invt_rows != nullptr && row_ok) ? ep.invt_rows[row] : ep.inv_temperature;
          const float sl2 = ep.invt_rows != nullptr ? it * 1.4426950408889634f : ep.scale_log2;
          constexpr int CPW = (BN / 32) / (EW / 4);  // 32-column chunks per warp
          const int cbeg = cgrp * CPW;
          // probability cache, 8-warp epilogue: the chunk's 16 packed fp16 pairs of every lane
          // (32 rows x 64 bytes) go through this warp's 2 KB staging buffer (64B swizzle,
          // conflict-free) and one TMA store; the global write leaves the drain's critical path
          [[maybe_unused]] auto p_stage_store = [&](int c, const uint32_t (&pk)[32]) {
            const uint32_t pbuf = smem_u32(sEpi) + 4096 + (warp - 2) * 2048;
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
  #pragma unroll
            for (int k = 0; k < 4; ++k)
              st_shared_v4(pbuf + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4), pk[4 * k], pk[4 * k + 1], pk[4 * k + 2],
                           pk[4 * k + 3]);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int c0 = n0 + c * 32;
              const int c1 = static_cast<int>(ep.p_row0) + m * TL::TILE_M + rank * 128 + q * 32;
              tma_store_2d(&tmC, sEpi + (pbuf - smem_u32(sEpi)), c0, c1);
              bulk_commit();
            }
          };
          // one 32-column chunk of scaled logits into the online (m, s, u) state and z_target
          auto lse_chunk = [&](int c, uint32_t (&r)[32]) {
            if (c * 32 >= nvalid) return;  // columns past V (ragged last tile)
#ifdef RL_AB_K1_NOMATH
            // A/B measurement only: read the accumulator, skip the softmax arithmetic
            if (r[0] == 0x7fc00001u) srun += 1.f;
            return;
#endif
            if (tl >= c * 32 && tl < c * 32 + 32) {
              const int jt = tl - c * 32;
              float z = -INFINITY;
  #pragma unroll
              for (int j = 0; j < 32; ++j) z = fmaxf(z, (j == jt) ? __uint_as_float(r[j]) : -INFINITY);
              zt = z * it;
            }
            if (c * 32 + 32 <= nvalid) {
              // full chunk: max on the raw accumulator (sl2 > 0) and the scale folded into one
              // FFMA per element (one ex2 per logit on the MUFU pipe, profiles/r02/k1_drain/)
              float cr = __uint_as_float(r[0]);
  #pragma unroll
              for (int j = 1; j < 32; ++j) cr = fmaxf(cr, __uint_as_float(r[j]));
              const float mn = fmaxf(mrun, cr * sl2);
              const float sc = ex2f(mrun - mn);
              trun = sc * fmaf(srun, mrun - mn, trun);
              srun *= sc;
              mrun = mn;
              if (ep.p_out == nullptr) {
  #pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const float d = fmaf(__uint_as_float(r[j]), sl2, -mn);
                  const float e = ex2f(d);
                  srun += e;
                  trun = fmaf(e, d, trun);
                }
                return;
              }
              // probability cache: the same exponentials, packed to fp16 pairs in place (r[j/2]
              // is rewritten only after r[j], r[j+1] are consumed) and stored with the chunk's m
  #pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float d0 = fmaf(__uint_as_float(r[j]), sl2, -mn);
                const float d1 = fmaf(__uint_as_float(r[j + 1]), sl2, -mn);
                const float e0 = ex2f(d0), e1 = ex2f(d1);
                srun += e0;
                trun = fmaf(e0, d0, trun);
                srun += e1;
                trun = fmaf(e1, d1, trun);
                r[j / 2] = pack_f16x2(e0, e1);
              }
              if constexpr (EW == 8) {
                if (ep.p_tma) {
                  p_stage_store(c, r);
                  if (row_ok) {
                    const int64_t col = static_cast<int64_t>(n0) + c * 32;
                    ep.p_m[(col >> 5) * ep.p_rows + ep.p_row0 + row] = mn;
                  }
                  return;
                }
              }
              if (row_ok) {
                const int64_t col = static_cast<int64_t>(n0) + c * 32;
                uint4* dst = reinterpret_cast<uint4*>(ep.p_out + (ep.p_row0 + row) * ep.p_ld + col);
                if (ep.p_evict_first) {
                  const uint64_t pol = l2_evict_first_policy();
  #pragma unroll
                  for (int k = 0; k < 4; ++k) st_global_v4_hint(dst + k, r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3], pol);
                } else {
  #pragma unroll
                  for (int k = 0; k < 4; ++k) dst[k] = make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
                }
                ep.p_m[(col >> 5) * ep.p_rows + ep.p_row0 + row] = mn;
              }
              return;
            }
            // the ragged last chunk of the vocabulary: columns past V are masked out
            float u[32];
  #pragma unroll
            for (int j = 0; j < 32; ++j) u[j] = (c * 32 + j < nvalid) ? __uint_as_float(r[j]) * sl2 : -1e30f;
            float cm = u[0];
  #pragma unroll
            for (int j = 1; j < 32; ++j) cm = fmaxf(cm, u[j]);
            const float mn = fmaxf(mrun, cm);
            const float sc = ex2f(mrun - mn);
            trun = sc * fmaf(srun, mrun - mn, trun);
            srun *= sc;
            mrun = mn;
  #pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float d = u[j] - mn;
              const float e = ex2f(d);
              srun += e;
              trun = fmaf(e, d, trun);
              u[j] = e;
            }
            if constexpr (EW == 8) {
              if (ep.p_out != nullptr && ep.p_tma) {  // TMA clips the columns past V
                uint32_t pk[32];
  #pragma unroll
                for (int j = 0; j < 16; ++j) pk[j] = pack_f16x2(u[2 * j], u[2 * j + 1]);
                p_stage_store(c, pk);
                if (row_ok) {
                  const int64_t col = static_cast<int64_t>(n0) + c * 32;
                  ep.p_m[(col >> 5) * ep.p_rows + ep.p_row0 + row] = mn;
                }
                return;
              }
            }
            if (ep.p_out != nullptr && row_ok) {  // probability cache: the valid columns only
              const int64_t col = static_cast<int64_t>(n0) + c * 32;
              uint16_t* dst = ep.p_out + (ep.p_row0 + row) * ep.p_ld + col;
              const int nv = nvalid - c * 32;
  #pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nv) dst[j] = f16_bits(u[j]);
              ep.p_m[(col >> 5) * ep.p_rows + ep.p_row0 + row] = mn;
            }
          };
          if constexpr (EW >= 8 && NB == 2 && CPW == 4) {
            // both TMEM halves of a wide tile through one 4-chunk register set: half 0 is loaded
            // and released at once; its arithmetic is split around the loads of half 1 (issued
            // into the slots already consumed), so half 1 goes back to the MMA after two
            // chunks of math instead of four (profiles/r02/k1_early_release/)
            if (h == 0) {
  #pragma unroll
              for (int k = 0; k < 4; ++k) tmem_ld32(taddr + (cbeg + k) * 32, lse_pre[k]);
              tmem_wait_ld();
              release_tmem(0);
              lse_chunk(cbeg + 0, lse_pre[0]);
              lse_chunk(cbeg + 1, lse_pre[1]);
              mbar_wait_sleep(&tfull[1], aph);
              tc_fence_after();
              const uint32_t taddr1 = taddr + BN;
              tmem_ld32(taddr1 + (cbeg + 0) * 32, lse_pre[0]);
              tmem_ld32(taddr1 + (cbeg + 1) * 32, lse_pre[1]);
              lse_chunk(cbeg + 2, lse_pre[2]);
              lse_chunk(cbeg + 3, lse_pre[3]);
              tmem_ld32(taddr1 + (cbeg + 2) * 32, lse_pre[2]);
              tmem_ld32(taddr1 + (cbeg + 3) * 32, lse_pre[3]);
              tmem_wait_ld();
              release_tmem(1);
            } else {
  #pragma unroll
              for (int k = 0; k < 4; ++k) lse_chunk(cbeg + k, lse_pre[k]);   // half 1, already loaded
            }
          } else if constexpr (EW >= 8) {
            // every chunk of this warp's share of the half in registers at once, then the TMEM
            // half goes back to the MMA: the softmax arithmetic (the drain's bottleneck) runs
            // under the next MMAs instead of in front of them
            uint32_t pre[CPW][32];
  #pragma unroll
            for (int k = 0; k < CPW; ++k) tmem_ld32(taddr + (cbeg + k) * 32, pre[k]);
            tmem_wait_ld();
            release_tmem(bi);
  #pragma unroll
            for (int k = 0; k < CPW; ++k) lse_chunk(cbeg + k, pre[k]);
          } else {
  #pragma unroll 1
            for (int c = cbeg; c < cbeg + CPW; ++c) {
              uint32_t r[32];
              tmem_ld32(taddr + c * 32, r);
              tmem_wait_ld();
              if (c == cbeg + CPW - 1) release_tmem(bi);
              lse_chunk(c, r);
            }
          }
          if constexpr (EW > 4) {
            // merge the column groups' states into group 0: (m, s, u) in log2 units, zt by
            // max, in group order (deterministic). Two slot sets used alternately: a set is
            // rewritten only after the barrier of the following merge, which the reading
            // warp reaches after reading it.
            constexpr int NG = EW / 4;
            float4* slots = reinterpret_cast<float4*>(sEpi) + ((merge_ctr++ & 1) * 4 + q) * (NG - 1) * 32 + lane;
            if (cgrp > 0) slots[(cgrp - 1) * 32] = make_float4(mrun, srun, trun, zt);
            named_bar_sync(1 + q, 32 * NG);
            if (cgrp > 0) continue;
  #pragma unroll
            for (int gi = 0; gi < NG - 1; ++gi) {
              const float4 o = slots[gi * 32];
              const float mn = fmaxf(mrun, o.x);
              const float a1 = ex2f(mrun - mn), a2 = ex2f(o.x - mn);
              trun = a1 * fmaf(srun, mrun - mn, trun) + a2 * fmaf(o.y, o.x - mn, o.z);
              srun = a1 * srun + a2 * o.y;
              mrun = mn;
              zt = fmaxf(zt, o.w);
            }
          }
          if (row_ok && n0 < ep.cols) {  // one partial per 256-column block
            constexpr float LN2 = 0.69314718055994530942f;
            ep.partials[static_cast<int64_t>(n * NB + h) * ep.rows + row] =
                make_float4(mrun * LN2, srun, trun * LN2, zt);
          }
        } else if (GROUPED && masked) {
          // masked per-row stores: rows past the group's end belong to the next group
          const int64_t cleft = ep.cols - n0;
          const int ncols = cleft < BN ? static_cast<int>(cleft) : BN;
          uint16_t* orow = ep.grouped_out + row * ep.cols + n0;
          const float rs = (ep.row_scale && row_ok) ? ep.row_scale[row] : 1.f;
  #pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(taddr + c * 32, r);
            tmem_wait_ld();
            if (c == BN / 32 - 1) release_tmem(bi);
            if (row_ok && c * 32 < ncols) {
              uint32_t w[16];
  #pragma unroll
              for (int j = 0; j < 16; ++j)
                w[j] = pack_bf16x2(__uint_as_float(r[2 * j]) * rs, __uint_as_float(r[2 * j + 1]) * rs);
              uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
  #pragma unroll
              for (int j = 0; j < 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            }
          }
        } else {
          // store epilogues: TMEM -> regs -> (math) -> swizzled smem -> TMA store
          float g = 0.f, b2 = 0.f, sl2 = ep.scale_log2;
          int tl = -1;
          const float rs = (GROUPED && ep.row_scale && row_ok) ? ep.row_scale[row] : 1.f;
          if constexpr (MODE == EPI_DZ) {
            if (row_ok) {
              const float it = ep.invt_rows != nullptr ? ep.invt_rows[row] : ep.inv_temperature;
              if (ep.invt_rows != nullptr) sl2 = it * 1.4426950408889634f;
              g = ep.coef[row] * it;
              b2 = ep.lse[row] * 1.4426950408889634f;
              const int64_t yl = static_cast<int64_t>(ep.targets[row]) - ep.vocab_offset;
              const int64_t t64 = yl - n0;
              tl = (yl < ep.cols && t64 >= 0 && t64 < BN) ? static_cast<int>(t64) : -1;
            }
          }
          constexpr int COLS = (MODE == EPI_DZ || MODE == EPI_BF16 || MODE == EPI_BF16_GROUPED) ? 64 : 32;
          // a tile with an empty K range (sparse backward, every row masked) stores zeros:
          // the MMA issued nothing, so TMEM holds no accumulator for it
          bool empty_k = false;
          if constexpr (!GROUPED) {
            int kb0, kb1;
            tile_k_range(tile, sh, kb0, kb1);
            empty_k = kb1 <= kb0;
          }
          if constexpr ((MODE == EPI_F32 || MODE == EPI_F32_ADD) && EW == 8) {
            // 8 warps, fp32 stores: a warp loads its 4 chunks of the half at once and releases
            // the TMEM half before storing any, so the next tile's MMAs never wait on stores
            constexpr int K8 = (BN / 32) / 2;
            const int sc0e = cgrp * K8;
            uint32_t pre[K8][32];
  #pragma unroll
            for (int k = 0; k < K8; ++k) tmem_ld32(taddr + (sc0e + k) * 32, pre[k]);
            tmem_wait_ld();
            release_tmem(bi);
  #pragma unroll
            for (int k = 0; k < K8; ++k) {
              if (empty_k) {
  #pragma unroll
                for (int j = 0; j < 32; ++j) pre[k][j] = 0u;
              }
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
              stage_row(buf0, lane, pre[k]);
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                const int c0 = n0 + (sc0e + k) * 32;
                const int c1 = m * TL::TILE_M + rank * 128 + q * 32 + (tile / (sh.m_blocks * sh.n_blocks)) * sh.split_rows;
                if (MODE == EPI_F32_ADD)
                  tma_reduce_add_2d(&tmC, sEpi + (buf0 - smem_u32(sEpi)), c0, c1);
                else
                  tma_store_2d(&tmC, sEpi + (buf0 - smem_u32(sEpi)), c0, c1);
                bulk_commit();
              }
              ++chunk_ctr;
            }
            continue;
          }
  #pragma unroll 1
          constexpr int SCPW = (BN / COLS) / (EW / 4);  // store chunks per warp and TMEM half
          const int sc0 = (MODE == EPI_LSE ? 0 : cgrp) * SCPW;
          for (int c = sc0; c < sc0 + SCPW; ++c) {
            uint32_t w[32];
            if constexpr (COLS == 64) {
              uint32_t r0[32], r1[32];
              tmem_ld32(taddr + c * 64, r0);
              tmem_ld32(taddr + c * 64 + 32, r1);
              tmem_wait_ld();
              if (c == sc0 + SCPW - 1) release_tmem(bi);
  #pragma unroll
              for (int j = 0; j < 16; ++j) {
                float v0 = __uint_as_float(r0[2 * j]), v1 = __uint_as_float(r0[2 * j + 1]);
                float v2 = __uint_as_float(r1[2 * j]), v3 = __uint_as_float(r1[2 * j + 1]);
                if constexpr (MODE == EPI_DZ) {
                  v0 = g * ex2f(fmaf(v0, sl2, -b2));
                  v1 = g * ex2f(fmaf(v1, sl2, -b2));
                  v2 = g * ex2f(fmaf(v2, sl2, -b2));
                  v3 = g * ex2f(fmaf(v3, sl2, -b2));
                  const int cb = c * 64;
                  if (tl == cb + 2 * j) v0 -= g;
                  if (tl == cb + 2 * j + 1) v1 -= g;
                  if (tl == cb + 32 + 2 * j) v2 -= g;
                  if (tl == cb + 32 + 2 * j + 1) v3 -= g;
                }
                if constexpr (GROUPED) {
                  v0 *= rs;
                  v1 *= rs;
                  v2 *= rs;
                  v3 *= rs;
                }
                w[j] = empty_k ? 0u : pack_bf16x2(v0, v1);
                w[16 + j] = empty_k ? 0u : pack_bf16x2(v2, v3);
              }
            } else {
              uint32_t r0[32];
              tmem_ld32(taddr + c * 32, r0);
              tmem_wait_ld();
              if (c == sc0 + SCPW - 1) release_tmem(bi);
  #pragma unroll
              for (int j = 0; j < 32; ++j) w[j] = empty_k ? 0u : r0[j];
            }
            if constexpr (MODE == EPI_F32_NVLS) {
              if (ep.row_map != nullptr) {
                // compacted rows: this thread's 128-byte piece of its row goes straight to
                // output row row_map[row] of the local replica
                const int64_t col = static_cast<int64_t>(n0) + c * 32;
                if (row < rows_valid && col < ep.cols) {
                  float* dst = ep.nvls_local + static_cast<int64_t>(ep.row_map[row]) * ep.cols + col;
                  if (col + 32 <= ep.cols) {
  #pragma unroll
                    for (int j = 0; j < 8; ++j)
                      reinterpret_cast<uint4*>(dst)[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
                  } else {
                    for (int j = 0; j < static_cast<int>(ep.cols - col); ++j) dst[j] = __uint_as_float(w[j]);
                  }
                }
                continue;
              }
            }
            const uint32_t buf = buf0 + (chunk_ctr % NBUF) * EPI_BUF_BYTES;
            if (lane == 0) bulk_wait_read<NBUF - 1>();
            __syncwarp();
            stage_row(buf, lane, w);
            fence_async_smem();
            __syncwarp();
#ifdef RL_AB_K4_NOSTORE
            // A/B measurement only (never in the product build): K4 without its dU write,
            // the math and the staging kept. The first K4 launch of the process stores, so
            // the dU buffer K5 / K6 read holds real values (the bench repeats one batch):
            // MMA power depends on the operand bits, and a never-written buffer is zeros
            if (MODE == EPI_DZ && ab_k4_skip) {
              ++chunk_ctr;
              continue;
            }
#endif
            if (lane == 0) {
              const int c0 = n0 + c * COLS;
              const int c1 = GROUPED ? tile_row0 + rank * 128 + q * 32
                                     : m * TL::TILE_M + rank * 128 + q * 32 +
                                           (tile / (sh.m_blocks * sh.n_blocks)) * sh.split_rows;
              if (MODE == EPI_F32_ADD || (MODE == EPI_F32_NVLS && ep.nvls_add))
                tma_reduce_add_2d(&tmC, sEpi + (buf - smem_u32(sEpi)), c0, c1);
              else
                tma_store_2d(&tmC, sEpi + (buf - smem_u32(sEpi)), c0, c1);
              bulk_commit();
            }
            ++chunk_ctr;
          }
        }
      }
      if constexpr (MODE == EPI_F32_NVLS) {
        // publish this warp's slab once its stores are globally visible
        if (ep.row_map != nullptr || ep.nvls_lag > 0) {
          if (ep.row_map != nullptr) fence_sys();  // every lane's plain row stores
          __syncwarp();
          if (lane == 0) {
            bulk_wait_all();
            fence_async_global();
            fence_sys();
            st_release_sys(ep.nvls_flags[ep.nvls_rank] + nvls_slab(tile, rank, q), ep.nvls_epoch);
          }
          __syncwarp();
          if (ep.nvls_lag > 0 && it >= ep.nvls_lag)
            nvls_reduce_slab(ep, sh, unit + (it - ep.nvls_lag) * n_units, rank, q, lane);
        } else if (it > 0) {
          // TMA stores with communication warps: publish the PREVIOUS tile's slab once
          // its bulk groups completed (all but this tile's kStoreGroups newest), so the
          // warp never blocks on the stores it just issued
          if (lane == 0) {
            bulk_wait<kStoreGroups>();
            fence_async_global();
            fence_sys();
            st_release_sys(ep.nvls_flags[ep.nvls_rank] + nvls_slab(tile - n_units, rank, q), ep.nvls_epoch);
          }
          __syncwarp();
        }
      }
      ++it;
      if (NACC == 2) acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if constexpr (MODE == EPI_F32_NVLS) {
      if (ep.nvls_lag > 0) {
        for (int j = it - ep.nvls_lag < 0 ? 0 : it - ep.nvls_lag; j < it; ++j)
          nvls_reduce_slab(ep, sh, unit + j * n_units, rank, q, lane);
      } else if (ep.row_map == nullptr && it > 0 && lane == 0) {
        bulk_wait_all();  // the last tile's slab
        fence_async_global();
        fence_sys();
        st_release_sys(ep.nvls_flags[ep.nvls_rank] + nvls_slab(unit + (it - 1) * n_units, rank, q), ep.nvls_epoch);
      }
      fence_sys();
    }
    if (lane == 0) bulk_wait_all();
    if (warp == 2 && lane == 0) {
      RL_AB_FLUSH(5);
      RL_AB_FLUSH(6);
    }
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
#ifdef RL_AB_K4_NOSTORE
  if (MODE == EPI_DZ && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_ab_k4_launches, 1u);
#endif
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc2(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace rl
