// SIMT kernels of the path: S0 advantages (K0), S2 partial merge (K2), S3 loss
// coefficients + report (K3a/K3b). All are memory/latency bound and tiny next to
// the GEMMs; reductions use fixed-order trees so results are bit-reproducible.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/rl.h"

namespace rl {

// ------------------------------------------------------------------- K0
// One warp per group: A = S - mean(S). Mean accumulated in fp64
// in index order by lane 0 (G is small: 16 in the paper's run).
__global__ void group_adv_kernel(const float* __restrict__ S, int num_groups, int G, float* __restrict__ A) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= num_groups) return;
  const float* s = S + static_cast<int64_t>(warp) * G;
  double sum = 0.0;
  if (lane == 0)
    for (int j = 0; j < G; ++j) sum += static_cast<double>(s[j]);
  sum = __shfl_sync(0xffffffffu, sum, 0);
  const double mean = sum / G;
  for (int j = lane; j < G; j += 32)
    A[static_cast<int64_t>(warp) * G + j] = static_cast<float>(static_cast<double>(s[j]) - mean);
}

// ------------------------------------------------------------------- K2
// Merge n_parts partials (m, s, u, zt) per row in index order. 256 threads =
// 64 rows x 4 slices; slice j takes parts j, j+4, ...; the 4 slice results are
// merged in slice order. Output either final (logprob, entropy, lse) or one
// merged float4 partial per row.
struct Part {
  float m, s, u, zt;
};
__device__ __forceinline__ Part merge2(Part a, Part b) {
  // m' = max; s' = s_a e^{m_a-m'} + s_b e^{m_b-m'};
  // u' = sum_x e^{m_x-m'} (u_x + s_x (m_x - m'));  zt' = max(zt)
  const float M = fmaxf(a.m, b.m);
  const float ea = (a.s > 0.f) ? expf(a.m - M) : 0.f;
  const float eb = (b.s > 0.f) ? expf(b.m - M) : 0.f;
  Part r;
  r.m = M;
  r.s = a.s * ea + b.s * eb;
  r.u = ea * (a.u + a.s * (a.m - M)) + eb * (b.u + b.s * (b.m - M));
  r.zt = fmaxf(a.zt, b.zt);
  return r;
}

// 32 rows x 8 vocab-tile slices per block (each warp reads 32 consecutive float4 of
// one tile: coalesced); 4 partial loads in flight per thread; slices combined by a
// fixed-order tree, so the merge order (and the result) does not depend on timing.
constexpr int MERGE_ROWS = 32, MERGE_SLICES = 8;
__global__ void __launch_bounds__(MERGE_ROWS * MERGE_SLICES)
    merge_partials_kernel(const float4* __restrict__ parts, int n_parts, int64_t T, float* __restrict__ logprob,
                          float* __restrict__ entropy, float* __restrict__ lse, float4* __restrict__ merged) {
  __shared__ Part sh[MERGE_SLICES][MERGE_ROWS];
  const int r = threadIdx.x % MERGE_ROWS;
  const int slice = threadIdx.x / MERGE_ROWS;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * MERGE_ROWS + r;
  Part acc = {-1e30f, 0.f, 0.f, -INFINITY};
  if (row < T) {
    int p = slice;
    for (; p + 3 * MERGE_SLICES < n_parts; p += 4 * MERGE_SLICES) {
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldg(parts + static_cast<int64_t>(p + k * MERGE_SLICES) * T + row);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc = merge2(acc, Part{v[k].x, v[k].y, v[k].z, v[k].w});
    }
    for (; p < n_parts; p += MERGE_SLICES) {
      const float4 v = __ldg(parts + static_cast<int64_t>(p) * T + row);
      acc = merge2(acc, Part{v.x, v.y, v.z, v.w});
    }
  }
  sh[slice][r] = acc;
  __syncthreads();
  if (slice == 0 && row < T) {
    Part a = merge2(merge2(merge2(sh[0][r], sh[1][r]), merge2(sh[2][r], sh[3][r])),
                    merge2(merge2(sh[4][r], sh[5][r]), merge2(sh[6][r], sh[7][r])));
    if (merged != nullptr) {
      merged[row] = make_float4(a.m, a.s, a.u, a.zt);
    } else {
      const float ls = logf(a.s);
      const float l = a.m + ls;
      logprob[row] = a.zt - l;
      if (entropy) entropy[row] = ls - a.u / a.s;
      if (lse) lse[row] = l;
    }
  }
}

// ------------------------------------------------------------------- K3
struct RolloutPartial {
  double loss;  // sum of coef over the rollout
  double kl;
  uint32_t kept, low, high, guarded, gtokens, nonfinite, badtgt, badoff;
};

template <typename T>
__device__ __forceinline__ T block_reduce_sum(T v, T* sh) {
  // fixed-order tree over blockDim.x (power of two) -> deterministic
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  T r = sh[0];
  __syncthreads();
  return r;
}

struct LossArgs {
  int variant;  // rl_loss_variant
  int kl_set;   // rl_kl_set
  double kl_w;  // kl_tau / D (reading R19); 0 = no KL term
  float alpha, beta, guard;
  double inv_D;
  int R;
  int64_t T;
  int64_t V_global;
  const float* logprob;
  const float* infer;
  const int32_t* targets;
  const float* adv;
  const int32_t* offsets;
  const uint8_t* loss_mask;
  float* coef;
  uint8_t* keep;
  uint8_t* guarded;
  RolloutPartial* rp;
  // rollouts split across ranks: the rollout statistics reduced over every
  // rank holding part of rollout i (rl_rollout_stats, then all-reduce MIN / SUM / SUM);
  // NULL = this call holds whole rollouts and computes them itself
  const float* ext_kmin;     // [R] min over valid tokens of k = exp(logprob - infer), +inf if none
  const double* ext_lr_sum;  // [R] sum over valid tokens of log k (GSPO)
  const int32_t* ext_n;      // [R] number of valid tokens (GSPO)
};

// A loss token that takes part in the loss and the guard: loss_mask, a finite stored
// log-prob <= 0 and (when targets are given) a target in [0, V_global).
__device__ __forceinline__ bool token_valid(const LossArgs& a, int64_t t) {
  const bool lm = a.loss_mask ? (a.loss_mask[t] != 0) : true;
  const float inf = a.infer[t];
  const bool fin = isfinite(inf) && inf <= 0.f;
  bool tg = true;
  if (a.targets) {
    const int32_t y = a.targets[t];
    tg = y >= 0 && static_cast<int64_t>(y) < a.V_global;
  }
  return lm && fin && tg;
}

// Per-rollout statistics of this rank's rows for rollouts split across ranks: one block
// per rollout, the same validity rule and fixed-order reductions as loss_coef_kernel.
__global__ void __launch_bounds__(256) rollout_stats_kernel(const LossArgs a, float* __restrict__ kmin_out,
                                                             double* __restrict__ lr_out, int32_t* __restrict__ n_out) {
  __shared__ double shd[256];
  __shared__ uint32_t shu[256];
  __shared__ float shf[256];
  const int i = blockIdx.x;
  int64_t t0 = a.offsets[i], t1 = a.offsets[i + 1];
  if (t0 < 0 || t1 > a.T || t1 < t0) t0 = t1 = 0;  // malformed offsets: counted by the loss call
  float kmin = INFINITY;
  double lr = 0.0;
  uint32_t n = 0;
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    if (token_valid(a, t)) {
      const float d = a.logprob[t] - a.infer[t];
      kmin = fminf(kmin, expf(d));
      lr += static_cast<double>(d);
      ++n;
    }
  }
  shf[threadIdx.x] = kmin;
  __syncthreads();
  for (int s2 = blockDim.x / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2) shf[threadIdx.x] = fminf(shf[threadIdx.x], shf[threadIdx.x + s2]);
    __syncthreads();
  }
  const double lr_all = block_reduce_sum(lr, shd);
  const uint32_t n_all = block_reduce_sum(n, shu);
  if (threadIdx.x == 0) {
    kmin_out[i] = shf[0];
    lr_out[i] = lr_all;
    n_out[i] = static_cast<int32_t>(n_all);
  }
}

// One block per rollout (256 threads). Pass 1: guard min over valid tokens.
// Pass 2: Eq.2 gate, coef, counters. Offsets are validated by every block so all
// blocks take the same decision without a grid-wide sync.
__global__ void __launch_bounds__(256) loss_coef_kernel(const LossArgs a) {
  __shared__ double shd[256];
  __shared__ uint32_t shu[256];
  __shared__ float shf[256];
  __shared__ int bad;
  const int i = blockIdx.x;
  if (threadIdx.x == 0) bad = (a.offsets[0] != 0 || a.offsets[a.R] != a.T) ? 1 : 0;
  __syncthreads();
  for (int j = threadIdx.x; j < a.R; j += blockDim.x)
    if (a.offsets[j] > a.offsets[j + 1]) bad = 1;
  __syncthreads();
  if (bad) {
    const int64_t t0 = a.T * i / a.R, t1 = a.T * (i + 1) / a.R;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
      a.coef[t] = 0.f;
      if (a.keep) a.keep[t] = 0;
    }
    if (threadIdx.x == 0) {
      if (a.guarded) a.guarded[i] = 0;
      RolloutPartial p = {};
      p.badoff = (i == 0) ? 1u : 0u;
      a.rp[i] = p;
    }
    return;
  }
  const int64_t t0 = a.offsets[i], t1 = a.offsets[i + 1];
  const double A = static_cast<double>(a.adv[i]);

  // pass 1: guard min over valid tokens (and, for GSPO, the mean log-ratio)
  float kmin = INFINITY;
  double lr_sum = 0.0;
  uint32_t n_valid = 0;
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    if (token_valid(a, t)) {
      const float d = a.logprob[t] - a.infer[t];
      kmin = fminf(kmin, expf(d));
      lr_sum += static_cast<double>(d);
      ++n_valid;
    }
  }
  // block min (fixed tree)
  shf[threadIdx.x] = kmin;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) shf[threadIdx.x] = fminf(shf[threadIdx.x], shf[threadIdx.x + s]);
    __syncthreads();
  }
  const bool g = (a.ext_kmin ? a.ext_kmin[i] : shf[0]) < a.guard;
  __syncthreads();
  // GSPO: s_i, the liveness and clip gate of the rollout (identical in every thread)
  float s_seq = 1.f, gspo_w = 0.f;
  bool gspo_live = false, gspo_clip_lo = false, gspo_clip_hi = false, gspo_u = false;
  double gspo_J = 0.0;
  if (a.variant == RL_LOSS_GSPO) {
    const double lr_local = block_reduce_sum(lr_sum, shd);
    const uint32_t n_local = block_reduce_sum(n_valid, shu);
    // split rollouts: s_i from the whole rollout; this rank adds its share n_local / n of J_i
    const double lr = a.ext_lr_sum ? a.ext_lr_sum[i] : lr_local;
    const uint32_t n = a.ext_n ? static_cast<uint32_t>(a.ext_n[i] > 0 ? a.ext_n[i] : 0) : n_local;
    const double share = (a.ext_n && n > 0) ? static_cast<double>(n_local) / n : 1.0;
    gspo_live = n > 0 && !g;
    s_seq = n > 0 ? static_cast<float>(exp(lr / n)) : 1.f;
    gspo_clip_hi = gspo_live && A > 0.0 && s_seq > a.beta;
    gspo_clip_lo = gspo_live && A < 0.0 && s_seq < a.alpha;
    gspo_u = gspo_live && !gspo_clip_hi && !gspo_clip_lo;
    gspo_w = gspo_u ? static_cast<float>(static_cast<double>(s_seq) * A / n * a.inv_D) : 0.f;
    if (gspo_live) {
      const double sc = fmin(fmax(static_cast<double>(s_seq), static_cast<double>(a.alpha)),
                             static_cast<double>(a.beta));
      gspo_J = fmin(static_cast<double>(s_seq) * A, sc * A) * a.inv_D * share;
    }
  }

  // pass 2: gate, coefficient, counters
  double loss = 0.0, kl = 0.0, klterm = 0.0;
  uint32_t kept = 0, low = 0, high = 0, gtok = 0, nonfin = 0, badtgt = 0;
  for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const bool lm = a.loss_mask ? (a.loss_mask[t] != 0) : true;
    const float inf = a.infer[t];
    const bool fin = isfinite(inf) && inf <= 0.f;
    bool tg = true;
    if (a.targets) {
      const int32_t y = a.targets[t];
      tg = y >= 0 && static_cast<int64_t>(y) < a.V_global;
    }
    const bool valid = lm && fin && tg;
    float c = 0.f;
    bool kp = false;
    if (valid) {
      const float lp = a.logprob[t];
      const float d = lp - inf;
      const float k = expf(d);
      gtok += g;
      kl += static_cast<double>(k) - static_cast<double>(d) - 1.0;
      if (a.variant == RL_LOSS_ICEPOP) {
        low += (k < a.alpha);
        high += (k > a.beta);
        kp = (k >= a.alpha) && (k <= a.beta) && !g;
        if (kp) {
          const double cd = static_cast<double>(k) * A * a.inv_D;
          c = static_cast<float>(cd);
          loss += cd;
        }
      } else if (a.variant == RL_LOSS_CISPO) {
        low += (k < a.alpha);
        high += (k > a.beta);
        kp = !g;
        if (kp) {
          const double cd = static_cast<double>(fminf(fmaxf(k, a.alpha), a.beta)) * A * a.inv_D;
          c = static_cast<float>(cd);
          loss += cd * static_cast<double>(lp);   // -loss = sum coef * logp
        }
      } else {  // GSPO
        low += gspo_clip_lo;
        high += gspo_clip_hi;
        kp = gspo_u;
        c = gspo_w;
      }
      kept += kp;
      if (a.kl_w != 0.0) {
        // R19: loss += (kl_tau/D) log k_t on the set S; coef_t -= kl_tau/D there
        const bool in_s = a.kl_set == RL_KL_ALL || (a.kl_set == RL_KL_UNMASKED ? kp : !kp);
        if (in_s) {
          klterm += a.kl_w * static_cast<double>(d);
          c = static_cast<float>(static_cast<double>(c) - a.kl_w);
        }
      }
    } else if (lm) {
      nonfin += !fin;
      badtgt += (fin && !tg);
    }
    a.coef[t] = c;
    if (a.keep) a.keep[t] = kp ? 1 : 0;
  }
  if (a.variant == RL_LOSS_GSPO) loss = (threadIdx.x == 0) ? gspo_J : 0.0;
  loss -= klterm;  // report.loss = -sum(loss): the KL term enters with a + sign
  RolloutPartial p;
  p.loss = block_reduce_sum(loss, shd);
  p.kl = block_reduce_sum(kl, shd);
  p.kept = block_reduce_sum(kept, shu);
  p.low = block_reduce_sum(low, shu);
  p.high = block_reduce_sum(high, shu);
  p.gtokens = block_reduce_sum(gtok, shu);
  p.nonfinite = block_reduce_sum(nonfin, shu);
  p.badtgt = block_reduce_sum(badtgt, shu);
  p.guarded = g ? 1u : 0u;
  p.badoff = 0;
  if (threadIdx.x == 0) {
    a.rp[i] = p;
    if (a.guarded) a.guarded[i] = g ? 1 : 0;
  }
}

// One block: sum the R rollout partials in index order -> report.
__global__ void loss_finalize_kernel(const RolloutPartial* __restrict__ rp, int R, rl_loss_report* rep) {
  if (threadIdx.x != 0) return;
  rl_loss_report r = {};
  double loss = 0.0, kl = 0.0;
  for (int i = 0; i < R; ++i) {
    const RolloutPartial p = rp[i];
    loss += p.loss;
    kl += p.kl;
    r.kept_tokens += p.kept;
    r.masked_low += p.low;
    r.masked_high += p.high;
    r.guarded_rollouts += p.guarded;
    r.guarded_tokens += p.gtokens;
    r.nonfinite_inputs += p.nonfinite;
    r.bad_targets += p.badtgt;
    r.bad_offsets += p.badoff;
  }
  r.loss = -loss;
  r.mismatch_kl_sum = kl;
  *rep = r;
}

// ------------------------------------------------- sparse backward (rows with coef != 0)
// Tokens whose coefficient is 0 (masked by Eq.2, guarded, loss_mask = 0, invalid)
// have an all-zero dU row: the backward GEMMs run on the compacted rows only.
// Compaction is order preserving and deterministic (block counts, then an in-block
// scan); counts per dU chunk go to chunk_counts[c] = clamp(count - c*chunk, 0, chunk).
constexpr int COMPACT_ROWS = 1024;  // rows per compaction block (256 threads x 4)

__global__ void compact_count_kernel(const float* __restrict__ coef, int64_t T, int* __restrict__ block_counts) {
  __shared__ int sh[256];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * COMPACT_ROWS + threadIdx.x * 4;
  int c = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) c += (r0 + j < T && coef[r0 + j] != 0.f) ? 1 : 0;
  const int tot = block_reduce_sum(c, sh);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

__global__ void compact_write_kernel(const float* __restrict__ coef, const float* __restrict__ lse,
                                     const int32_t* __restrict__ targets, int64_t T,
                                     const int* __restrict__ block_counts, int nblocks, int64_t chunk,
                                     int32_t* __restrict__ idx, float* __restrict__ coef_c, float* __restrict__ lse_c,
                                     int32_t* __restrict__ tgt_c, int* __restrict__ chunk_counts, int n_chunks,
                                     const float* __restrict__ invt_rows, float* __restrict__ invt_c) {
  __shared__ int sh[256];
  __shared__ int base;
  if (threadIdx.x == 0) {
    int b = 0;
    for (int j = 0; j < static_cast<int>(blockIdx.x); ++j) b += block_counts[j];
    base = b;
  }
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * COMPACT_ROWS + threadIdx.x * 4;
  bool f[4];
  int c = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[j] = r0 + j < T && coef[r0 + j] != 0.f;
    c += f[j];
  }
  // exclusive scan of c over the block (Hillis-Steele in shared memory)
  sh[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int v = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += v;
    __syncthreads();
  }
  int pos = base + sh[threadIdx.x] - c;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (f[j]) {
      const int64_t r = r0 + j;
      idx[pos] = static_cast<int32_t>(r);
      coef_c[pos] = coef[r];
      lse_c[pos] = lse[r];
      tgt_c[pos] = targets[r];
      if (invt_rows != nullptr) invt_c[pos] = invt_rows[r];
      ++pos;
    }
  if (blockIdx.x == nblocks - 1 && threadIdx.x == 255) {
    const int64_t count = pos;  // = base + inclusive scan of the last thread
    for (int ch = 0; ch < n_chunks; ++ch) {
      const int64_t left = count - ch * chunk;
      chunk_counts[ch] = static_cast<int>(left < 0 ? 0 : (left > chunk ? chunk : left));
    }
    chunk_counts[n_chunks] = static_cast<int>(count);
  }
}

// h_c[r] = hidden[idx[r]] for r < count; the `pad` rows after them (up to `cap`) are
// zeroed together with their coef/lse/target, so a tail tile of any chunk (which
// reads at most 255 rows past the chunk's last compact row) contributes exact zeros.
// Flat over (row, 16-byte vector), 4 loads in flight per thread before the stores.
__global__ void gather_rows_kernel(const uint16_t* __restrict__ hidden, int64_t H, const int32_t* __restrict__ idx,
                                   const int* __restrict__ count_ptr, int pad, int64_t cap, uint16_t* __restrict__ h_c,
                                   float* __restrict__ coef_c, float* __restrict__ lse_c, int32_t* __restrict__ tgt_c,
                                   float* __restrict__ invt_c) {
  const int count = *count_ptr;
  const int64_t padded = (static_cast<int64_t>(count) + pad < cap) ? static_cast<int64_t>(count) + pad : cap;
  const int64_t vecs = H / 8;  // 16-byte vectors per row (H % 8 == 0)
  const int64_t n = padded * vecs;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(hidden);
  uint4* dst = reinterpret_cast<uint4*>(h_c);
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + k * stride;
      v[k] = make_uint4(0, 0, 0, 0);
      if (i < n) {
        const int64_t r = i / vecs;
        if (r < count) v[k] = __ldg(src + static_cast<int64_t>(idx[r]) * vecs + (i - r * vecs));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + k * stride;
      if (i < n) {
        dst[i] = v[k];
        const int64_t r = i / vecs;
        if (r >= count && i == r * vecs) {
          coef_c[r] = 0.f;
          lse_c[r] = 0.f;
          tgt_c[r] = -1;
          if (invt_c != nullptr) invt_c[r] = 1.f;
        }
      }
    }
  }
}

// dh[idx[r]] = dh_c[r] for r < count (dh pre-zeroed); row_bytes % 16 == 0.
__global__ void scatter_rows_kernel(const uint8_t* __restrict__ dh_c, int64_t row_bytes,
                                    const int32_t* __restrict__ idx, const int* __restrict__ count_ptr,
                                    uint8_t* __restrict__ dh) {
  const int count = *count_ptr;
  const int64_t vecs = row_bytes / 16;
  const int64_t n = static_cast<int64_t>(count) * vecs;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(dh_c);
  uint4* dst = reinterpret_cast<uint4*>(dh);
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + k * stride;
      if (i < n) v[k] = __ldg(src + i);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = i0 + k * stride;
      if (i < n) {
        const int64_t r = i / vecs;
        dst[static_cast<int64_t>(idx[r]) * vecs + (i - r * vecs)] = v[k];
      }
    }
  }
}

// ------------------------------------------------------- Newton-Schulz aux
// Frobenius norm: per-block fp64 partial sums of squares (fixed order), then every
// block of the cast kernel re-sums the partials in index order (deterministic).
__global__ void sumsq_partial_kernel(const float* __restrict__ g, int64_t n, double* __restrict__ partials) {
  __shared__ double sh[256];
  // 128-bit loads, 4 independent fp32 squares per load folded into one fp64 accumulator
  double acc = 0.0;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = g4[i];
    acc += static_cast<double>(v.x * v.x + v.y * v.y) + static_cast<double>(v.z * v.z + v.w * v.w);
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = g[i];
    acc += v * v;
  }
  const double tot = block_reduce_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// X_0 = bf16(g / (||g||_F + eps)); optionally u = g + mu*m first (Muon, fused).
__global__ void ns_prep_kernel(const float* __restrict__ g, int64_t n, const double* __restrict__ partials,
                               int nparts, uint16_t* __restrict__ x0) {
  // every block re-sums the partials with the same fixed-order tree -> identical norms
  __shared__ double sh[256];
  double part = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) part += partials[i];
  const double tot = block_reduce_sum(part, sh);
  const float s = static_cast<float>(1.0 / (sqrt(tot) + 1e-7));
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint2* x4 = reinterpret_cast<uint2*>(x0);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = g4[i];
    uint2 o;
    o.x = static_cast<uint32_t>(f32_to_bf16_bits(v.x * s)) | (static_cast<uint32_t>(f32_to_bf16_bits(v.y * s)) << 16);
    o.y = static_cast<uint32_t>(f32_to_bf16_bits(v.z * s)) | (static_cast<uint32_t>(f32_to_bf16_bits(v.w * s)) << 16);
    x4[i] = o;
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    x0[i] = f32_to_bf16_bits(g[i] * s);
}

// out[0] = fixed-order sum of n fp64 partials (one block)
__global__ void sum_partials_kernel(const double* __restrict__ partials, int n, double* __restrict__ out) {
  __shared__ double sh[256];
  double p = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) p += partials[i];
  const double t = block_reduce_sum(p, sh);
  if (threadIdx.x == 0) out[0] = t;
}

__global__ void cast_bf16_kernel(const float* __restrict__ a, int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f32_to_bf16_bits(a[i]);
}

// Split-K reduction in index order (deterministic): out32 = sum_s parts[s], out16 = bf16(out32).
__global__ void split_reduce_cast_kernel(const float* __restrict__ parts, int splits, int64_t n,
                                         float* __restrict__ out32, uint16_t* __restrict__ out16) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = parts[i];
    for (int s = 1; s < splits; ++s) acc += parts[static_cast<int64_t>(s) * n + i];
    out32[i] = acc;
    out16[i] = f32_to_bf16_bits(acc);
  }
}

// C = bf16(a I + b A + c A2) for K x K matrices.
__global__ void ns_poly_kernel(const float* __restrict__ A, const float* __restrict__ A2, int64_t K, float ca,
                               float cb, float cc, uint16_t* __restrict__ C) {
  const int64_t n = K * K;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float diag = (i / K == i % K) ? ca : 0.f;
    C[i] = f32_to_bf16_bits(diag + cb * A[i] + cc * A2[i]);
  }
}

// Muon momentum: m <- mu m + g; u = nesterov ? g + mu m : m (fp32, in place on m, u out).
__global__ void muon_momentum_kernel(const float* __restrict__ g, float* __restrict__ m, float* __restrict__ u,
                                     int64_t n, float mu, int nesterov) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float mi = mu * m[i] + g[i];
    m[i] = mi;
    u[i] = nesterov ? g[i] + mu * mi : mi;
  }
}

// theta <- theta (1 - lr wd) - lr * scale * O  (O bf16 from Newton-Schulz).
__global__ void muon_apply_kernel(float* __restrict__ theta, const uint16_t* __restrict__ o, int64_t n, float decay,
                                  float step) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    theta[i] = theta[i] * decay - step * __bfloat162float(__ushort_as_bfloat16(o[i]));
}

// 1 / sqrt(mean_k x[r, k]^2 + eps) per row (bf16 x), one warp per row, fixed-order sums.
__global__ void rms_inv_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t K, float eps,
                               float* __restrict__ out) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const uint16_t* xr = x + r * K;
  float acc = 0.f;
  for (int64_t k = lane; k < K; k += 32) {
    const float v = __bfloat162float(__ushort_as_bfloat16(xr[k]));
    acc = fmaf(v, v, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[r] = rsqrtf(acc / static_cast<float>(K) + eps);
}


// out[r, k] = bf16(w[r, k] * gamma[k]): the RMSNorm weight folded into the expert weights
// along K (once per optimizer step), so the expert GEMM of RMSNorm(x) needs only the
// 1/rms row scale in its epilogue. 8 bf16 (16 B) per thread and iteration, grid-stride.
__global__ void fold_gamma_kernel(const uint16_t* __restrict__ w, const float* __restrict__ gamma, int64_t rows,
                                  int64_t K, uint16_t* __restrict__ out) {
  const int64_t n8 = rows * K / 8;  // K % 8 == 0
  const int64_t k8 = K / 8;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(w)[i];
    const int64_t k0 = (i % k8) * 8;
    const float4 g0 = *reinterpret_cast<const float4*>(gamma + k0);
    const float4 g1 = *reinterpret_cast<const float4*>(gamma + k0 + 4);
    const float gs[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const uint32_t in[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __uint_as_float(in[j] << 16) * gs[2 * j];
      const float hi = __uint_as_float(in[j] & 0xffff0000u) * gs[2 * j + 1];
      o[j] = pack_bf16x2(lo, hi);
    }
    reinterpret_cast<uint4*>(out)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Expert-load statistics from the device group offsets: out[0] = max_g load,
// out[1] = mean load, out[2] = MaxViolation = (max - mean) / mean (0 when there are no
// rows). One block; a group's load is its row count as the grouped GEMM sees it (offsets
// clamped to [0, rows], an end below its begin counts as empty).
__device__ __forceinline__ int64_t group_load(const int32_t* offsets, int g, int64_t rows) {
  const int64_t b = min(max(static_cast<int64_t>(offsets[g]), int64_t(0)), rows);
  const int64_t e = min(max(static_cast<int64_t>(offsets[g + 1]), int64_t(0)), rows);
  return e > b ? e - b : 0;
}

__global__ void expert_load_kernel(const int32_t* __restrict__ offsets, int n_groups, int64_t rows,
                                   float* __restrict__ out) {
  __shared__ long long smax[32], ssum[32];
  long long mx = 0, sum = 0;
  for (int g = threadIdx.x; g < n_groups; g += blockDim.x) {
    const long long l = group_load(offsets, g, rows);
    mx = max(mx, l);
    sum += l;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    smax[threadIdx.x >> 5] = mx;
    ssum[threadIdx.x >> 5] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x + 31) / 32; ++w) {
      mx = max(mx, smax[w]);
      sum += ssum[w];
    }
    const double mean = static_cast<double>(sum) / n_groups;
    out[0] = static_cast<float>(mx);
    out[1] = static_cast<float>(mean);
    out[2] = mean > 0 ? static_cast<float>((static_cast<double>(mx) - mean) / mean) : 0.f;
  }
}


// Split-K dH (few output tiles): out[r, :] = sum_s part[s * rows_pad + r, :] in split order
// (deterministic), for r < rows (or the device row count); bf16 (RN) or fp32 output.
template <typename OutT>
__global__ void split_sum_kernel(const float* __restrict__ part, int S, int64_t rows_pad, int64_t H, int64_t rows,
                                 const int* __restrict__ cnt, OutT* __restrict__ out) {
  int64_t n = rows;
  if (cnt) {
    const int64_t c = *cnt;
    n = c < rows ? (c > 0 ? c : 0) : rows;
  }
  const int64_t n4 = n * H / 4, stride4 = rows_pad * H / 4;
  const float4* p = reinterpret_cast<const float4*>(part);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = p[i];
    for (int k = 1; k < S; ++k) {
      const float4 b = p[k * stride4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    if constexpr (sizeof(OutT) == 2) {
      reinterpret_cast<uint2*>(out)[i] = make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w));
    } else {
      reinterpret_cast<float4*>(out)[i] = a;
    }
  }
}

// K4 from the probability cache (S4 without the recompute GEMM; EpiParams::p_out): for
// row i < n (n = *cnt when given) and column v < V,
//   dU[i, v] = bf16(g_i 2^(m[t, v/32] - lse_i log2 e) p~[t, v] - [v == y_i] g_i),  g_i = coef_i invT_i,
// the same value K4 computes as g_i 2^(z sl2 - lse_i log2 e) - [v == y_i] g_i, with t = row_map[i]
// (compacted rows) or row0 + i; coef / lse / targets / invt are indexed by i. Rows n .. up to the
// next multiple of 256 (at most `rows`) are written as zeros, as K4 does: K6 reads whole 64-row
// k-blocks past the device row count. HBM-bound: 2 B read + 2 B written per element. One block
// per row at a time (grid-stride over rows): each thread moves 16-byte vectors 256 apart, so
// every warp instruction covers 512 contiguous bytes of the row; DZC_UNROLL vectors in flight.
constexpr int DZC_THREADS = 256, DZC_UNROLL = 4;
__global__ void __launch_bounds__(DZC_THREADS) dz_from_cache_kernel(
    const uint16_t* __restrict__ pc, const float* __restrict__ pm, int64_t ld, int64_t p_rows,
    const int32_t* __restrict__ row_map, int64_t row0, const int* __restrict__ cnt, int64_t rows, int64_t V,
    const float* __restrict__ coef, const float* __restrict__ lse, const int32_t* __restrict__ targets,
    int64_t vocab_offset, const float* __restrict__ invt_rows, float inv_temperature, uint16_t* __restrict__ dz) {
  int64_t n = rows;
  if (cnt) {
    const int64_t c = *cnt;
    n = c < rows ? (c > 0 ? c : 0) : rows;
  }
  const int64_t n_pad = (n + 255) / 256 * 256 < rows ? (n + 255) / 256 * 256 : rows;
  const int nvec = static_cast<int>(V / 8);  // full 8-column vectors per row
  for (int64_t i = blockIdx.x; i < n_pad; i += gridDim.x) {
    uint16_t* drow = dz + i * ld;
    if (i >= n) {  // padding rows of the last 256-row block
      for (int k = threadIdx.x; k < nvec; k += DZC_THREADS) reinterpret_cast<uint4*>(drow)[k] = make_uint4(0u, 0u, 0u, 0u);
      for (int64_t v = static_cast<int64_t>(nvec) * 8 + threadIdx.x; v < V; v += DZC_THREADS) drow[v] = 0;
      continue;
    }
    const int64_t t = row_map ? static_cast<int64_t>(row_map[i]) : row0 + i;
    const float g = coef[i] * (invt_rows ? invt_rows[i] : inv_temperature);
    const float b2 = lse[i] * 1.4426950408889634f;
    const int64_t y = static_cast<int64_t>(targets[i]) - vocab_offset;
    const uint16_t* prow = pc + t * ld;
    const float* mrow = pm + t;
    auto one = [&](int k, const uint4 p) {
      const int64_t v0 = static_cast<int64_t>(k) * 8;
      const float sc = g * ex2f(mrow[(v0 >> 5) * p_rows] - b2);
      const uint32_t w[4] = {p.x, p.y, p.z, p.w};
      uint32_t o[4];
  #pragma unroll
      for (int q = 0; q < 4; ++q) {
        float a = sc * f16_to_f32(static_cast<uint16_t>(w[q] & 0xffffu));
        float b = sc * f16_to_f32(static_cast<uint16_t>(w[q] >> 16));
        if (y == v0 + 2 * q) a -= g;
        if (y == v0 + 2 * q + 1) b -= g;
        o[q] = pack_bf16x2(a, b);
      }
      reinterpret_cast<uint4*>(drow)[k] = make_uint4(o[0], o[1], o[2], o[3]);
    };
    int k = threadIdx.x;
    for (; k + (DZC_UNROLL - 1) * DZC_THREADS < nvec; k += DZC_UNROLL * DZC_THREADS) {
      uint4 p[DZC_UNROLL];
  #pragma unroll
      for (int u = 0; u < DZC_UNROLL; ++u) p[u] = reinterpret_cast<const uint4*>(prow)[k + u * DZC_THREADS];
  #pragma unroll
      for (int u = 0; u < DZC_UNROLL; ++u) one(k + u * DZC_THREADS, p[u]);
    }
    for (; k < nvec; k += DZC_THREADS) one(k, reinterpret_cast<const uint4*>(prow)[k]);
    for (int64_t v = static_cast<int64_t>(nvec) * 8 + threadIdx.x; v < V; v += DZC_THREADS) {  // ragged tail
      float a = g * ex2f(mrow[(v >> 5) * p_rows] - b2) * f16_to_f32(prow[v]);
      if (y == v) a -= g;
      drow[v] = static_cast<uint16_t>(pack_bf16x2(a, 0.f) & 0xffffu);
    }
  }
}

}  // namespace rl
