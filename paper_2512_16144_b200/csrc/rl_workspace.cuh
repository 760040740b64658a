// librl host code: workspace layout and host-side argument checks.
// Included once, in order, by rl_api.cu (a single translation unit); everything
// here has internal linkage.
#pragma once

namespace {

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
  // split-K dH for chunks with fewer 256 x 512 output tiles than CTA pairs: fp32 partials
  size_t dh_split;
  int dh_splits;
  int64_t n_tiles_v, ldz, chunk;
  // probability cache (fused step): K1 writes fp16 2^(z sl2 - m) [T x ldz]
  // and the per-32-column m [ceil(V/32) x T]; K4 then reads it instead of recomputing z
  size_t pc, pm;
  bool pcache;
};

// RL_P_CACHE = 0/1 (default 1): cache the softmax numerators in K1 so the fused step's K4 is an
// elementwise pass instead of a second LM-head GEMM. The workspace grows by
// T x V x 2 + T x V / 8 bytes (the whole batch, also when dU is processed in chunks).
// RL_P_EVICT = 0/1 (default 0): K1's direct (non-TMA) cache stores with an L2 evict-first policy;
// measured neutral (DRAM reads 6.98 vs 6.92 GB, same cycles; profiles/r02/pcache/pevict/).
bool pcache_evict_first() {
  static const int v = [] {
    const char* e = getenv("RL_P_EVICT");
    return e ? atoi(e) : 0;
  }();
  return v != 0;
}
// RL_P_TMA = 0/1 (default 1): the 8-warp K1 epilogue stages each cached chunk in shared memory and
// TMA-stores it (0: direct 16-byte global stores from the registers).
bool pcache_tma() {
  static const int v = [] {
    const char* e = getenv("RL_P_TMA");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}
bool pcache_enabled() {
  static const int v = [] {
    const char* e = getenv("RL_P_CACHE");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// K5 (dH = dU W, K = V) has only ceil(rows/256) x ceil(H/512) output tiles: with fewer than
// a B200's 74 CTA pairs the GEMM leaves pairs idle for a whole (long) tile. Split the
// vocabulary S ways (fp32 partials, summed in a fixed order) with the S in 2..8 that
// minimises the waves per unit of work, when that saves at least a quarter (the partials
// cost an extra S x rows x H x 8 bytes: at 2048 rows x 4096 an 8-way split measured slower,
// profiles/r02/dh_split/); 1 otherwise.
int dh_split_factor(int64_t rows, int64_t H, int64_t V) {
  constexpr int kPairs = 74;
  const int64_t tiles = ((rows + 255) / 256) * ((H + 511) / 512);
  if (rows <= 0 || tiles >= kPairs) return 1;
  int best_s = 1;
  double best = 1.0;
  for (int sp = 2; sp <= 8; ++sp) {
    if (V < int64_t(sp) * 64 * 16) break;  // keep >= 16 k-blocks per split
    const double t = static_cast<double>((tiles * sp + kPairs - 1) / kPairs) / sp;
    if (t < best - 1e-9) {
      best = t;
      best_s = sp;
    }
  }
  return best <= 0.75 ? best_s : 1;
}

int64_t n_vocab_tiles(const rl_lm_shape* s) { return (s->V_local + rl::BN - 1) / rl::BN; }

WsLayout ws_layout(const rl_lm_shape* s, int32_t R, int64_t chunk_rows) {
  WsLayout w;
  Carve c;
  const int64_t T = s->T > 0 ? s->T : 0;
  w.n_tiles_v = n_vocab_tiles(s);
  w.ldz = (s->V_local + 7) / 8 * 8;
  w.chunk = (chunk_rows <= 0 || chunk_rows > T) ? T : chunk_rows;
  // the probability cache first: its offset depends on T and V only, so a split-phase forward
  // (rl_fwd_partials_ex) and backward (rl_bwd_ex) with different dz_chunk_rows agree on it
  // the cache holds the whole batch (K4 fills each dU chunk from its rows); at most 64 GB
  w.pcache = pcache_enabled() && T > 0 && static_cast<double>(T) * w.ldz * 2.125 <= 64e9;
  w.pc = c.take(w.pcache ? static_cast<size_t>(T) * w.ldz * 2 : 0);
  w.pm = c.take(w.pcache ? static_cast<size_t>((s->V_local + 31) / 32) * T * 4 : 0);
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
  w.dh_splits = dh_split_factor(w.chunk, s->H, s->V_local);
  w.dh_split = c.take(w.dh_splits > 1 ? static_cast<size_t>(w.dh_splits) * ((w.chunk + 255) / 256 * 256) * s->H * 4
                                      : 0);
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
static_assert(sizeof(rl_nvls_reduce) == 96, "rl_nvls_reduce layout (binding mirrors it)");

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

}  // namespace
