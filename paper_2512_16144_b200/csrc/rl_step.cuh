// librl host code: the step phases: forward (K1+K2), loss (K3), NVLS descriptors, dense and sparse backward (K4-K6).
// Included once, in order, by rl_api.cu (a single translation unit); everything
// here has internal linkage.
#pragma once

namespace {

// K1 (+ K2): forward over the local shard. If `merged` is non-null, write one
// merged partial per row; else write logprob/entropy/lse.
// pc_rows > 0: also fill the probability cache (rows pc_row0 .. of a batch of pc_rows).
rl_status forward_impl(const rl_lm_shape* s, const uint16_t* hidden, const uint16_t* w, const int32_t* targets,
                       float* logprob, float* entropy, float* lse, float4* merged, uint8_t* ws, const WsLayout& L,
                       int sms, cudaStream_t st, int64_t pc_row0 = 0, int64_t pc_rows = 0) {
  const int64_t T = s->T;
  if (T == 0) return RL_OK;
  CUtensorMap ta, tb, tp;
  RL_TRY(make_map(&ta, hidden, false, s->H, T, s->H, 64, kARows));
  RL_TRY(make_map(&tb, w, false, s->H, s->V_local, s->H, 64, rl::BN / cta_group()));
  tp = ta;
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
  if (pc_rows > 0 && L.pcache) {
    ep.p_out = reinterpret_cast<uint16_t*>(ws + L.pc);
    ep.p_m = reinterpret_cast<float*>(ws + L.pm);
    ep.p_ld = L.ldz;
    ep.p_row0 = pc_row0;
    ep.p_rows = pc_rows;
    ep.p_evict_first = pcache_evict_first() ? 1 : 0;
    // 32 x 32 fp16 boxes (64-byte rows, 64B swizzle) for the TMA stores of the 8-warp epilogue
    if (pcache_tma()) {
      RL_TRY(make_map(&tp, ws + L.pc, false, s->V_local, pc_rows, L.ldz, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B));
      ep.p_tma = 1;
    }
  }
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + L.sync);
  RL_TRY((launch_gemm<rl::EPI_LSE, false, false>(RL_K_FWD_GEMM, ta, tb, tp, T, s->V_local, s->H, group_m_for(RL_K_FWD_GEMM, 16), ep, sms, st)));
  const int blocks = static_cast<int>((T + rl::MERGE_ROWS - 1) / rl::MERGE_ROWS);
  {
    ProfScope ps(RL_K_MERGE, st);
    rl::merge_partials_kernel<<<blocks, 256, 0, st>>>(parts, static_cast<int>(L.n_tiles_v), T, logprob, entropy,
                                                        lse, merged);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl::LossArgs loss_args(const rl_loss_params* p, int64_t T, int64_t V_global, const float* logprob,
                       const float* infer, const int32_t* targets, const float* adv, const int32_t* offsets,
                       const uint8_t* loss_mask) {
  rl::LossArgs a = {};
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
  return a;
}

rl_status loss_impl(const rl_loss_params* p, int64_t T, int64_t V_global, const float* logprob, const float* infer,
                    const int32_t* targets, const float* adv, const int32_t* offsets, const uint8_t* loss_mask,
                    float* coef, uint8_t* keep, uint8_t* guarded, rl_loss_report* rep, rl::RolloutPartial* rp,
                    cudaStream_t st, const float* ext_kmin = nullptr, const double* ext_lr_sum = nullptr,
                    const int32_t* ext_n = nullptr) {
  rl::LossArgs a = loss_args(p, T, V_global, logprob, infer, targets, adv, offsets, loss_mask);
  a.coef = coef;
  a.keep = keep;
  a.guarded = guarded;
  a.rp = rp;
  a.ext_kmin = ext_kmin;
  a.ext_lr_sum = ext_lr_sum;
  a.ext_n = ext_n;
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
int64_t nvls_shard_rows(int64_t rows, int32_t world) {
  return world > 0 ? (rows + 32 * int64_t(world) - 1) / (32 * int64_t(world)) * 32 : rows;
}

// e.rows must be set first (the reduce-scatter shard is a row range of D).
// `local` is this rank's replica at D's row 0 and `mc_off` the same offset (in
// floats) into the multicast VA. Each call's flags carry epoch * 256 + chunk, so
// epochs increase from chunk to chunk and from call to call (rl_nvls_reduce.epoch
// < 2^24, at most 256 chunks per call).
constexpr int kNvlsChunkEpochs = 256;
void set_nvls(rl::EpiParams& e, const rl_nvls_reduce* n, float* local, int64_t mc_off = 0, int chunk = 0) {
  e.nvls_local = local;
  e.nvls_mode = n->mode;
  e.nvls_shard = nvls_shard_rows(e.rows, n->world);
  e.nvls_mc = static_cast<float*>(n->multicast) + mc_off;
  for (int r = 0; r < rl::NVLS_MAX_RANKS; ++r) e.nvls_flags[r] = n->flags[r];
  e.nvls_rank = n->rank;
  e.nvls_world = n->world;
  e.nvls_epoch = n->epoch * kNvlsChunkEpochs + static_cast<uint32_t>(chunk);
  e.nvls_lag = n->lag > 0 ? n->lag : 0;  // 0: communication warps (default)
}

rl_status check_nvls(const rl_nvls_reduce* n, const char* what) {
  if (!n) return RL_OK;
  if (!n->multicast) return fail(RL_ERR_INVALID_ARGUMENT, "%s: multicast VA is NULL", what);
  if (n->world < 2 || n->world > RL_NVLS_MAX_RANKS || n->rank < 0 || n->rank >= n->world)
    return fail(RL_ERR_INVALID_ARGUMENT, "%s: need 2 <= world <= %d and 0 <= rank < world", what, RL_NVLS_MAX_RANKS);
  for (int r = 0; r < n->world; ++r)
    if (!n->flags[r]) return fail(RL_ERR_INVALID_ARGUMENT, "%s: flags[%d] is NULL", what, r);
  if (n->epoch == 0 || n->epoch >= (1u << 24))
    return fail(RL_ERR_INVALID_ARGUMENT, "%s: need 0 < epoch < 2^24 (flags start at 0)", what);
  if (n->mode != RL_NVLS_ALL_REDUCE && n->mode != RL_NVLS_REDUCE_SCATTER)
    return fail(RL_ERR_INVALID_ARGUMENT, "%s: unknown mode %d", what, n->mode);
  return RL_OK;
}

// K6 of the last dU chunk, with the NVLS dW reduction fused: adds to d_w_vocab when it
// already holds earlier chunks or micro-batches (`add`). With K = 0 (a rank with no
// rows) the epilogue stores zeros (or adds nothing) and still takes part in the
// reduction of every slab, so the other ranks never wait for it.
rl_status launch_dw_nvls(const CUtensorMap& t_dz_mn, const CUtensorMap& t_h_mn, const CUtensorMap& t_dw, int64_t V,
                         int64_t H, int64_t K, float* dw, const rl_nvls_reduce* n, bool add, int sms, cudaStream_t st,
                         const int* dyn_count = nullptr) {
  rl::EpiParams e6 = {};
  e6.rows = V;
  e6.cols = H;
  set_nvls(e6, n, dw);
  e6.nvls_add = add ? 1 : 0;
  return launch_gemm<rl::EPI_F32_NVLS, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, K,
                                                    group_m_for(RL_K_DW_GEMM, kGroupMBwd), e6, sms, st, 1, 0,
                                                    dyn_count, dyn_count ? 2 : 0);
}

// K5 (dH = dU W) for `rows` rows into `out` (bf16 or fp32, row-major [rows, H]); `cnt` (device,
// optional) is the actual row count of a compacted chunk. With fewer output tiles than CTA pairs
// (L.dh_splits > 1) the vocabulary is split: fp32 partials per split, then a fixed-order sum.
rl_status launch_dh(const CUtensorMap& t_dz_k, const CUtensorMap& t_w_mn, int64_t rows, int64_t H, int64_t V,
                    void* out, bool bf16_out, const int* cnt, uint8_t* ws, const WsLayout& L, int sms, cudaStream_t st) {
  rl::EpiParams e5 = {};
  e5.rows = rows;
  e5.cols = H;
  const int dyn = cnt ? 1 : 0;
  const int S = L.dh_splits;
  if (S <= 1 || dh_split_factor(rows, H, V) <= 1) {
    CUtensorMap t_dh;
    if (bf16_out) {
      RL_TRY(make_map(&t_dh, out, false, H, rows, H, 64, 32));
      return launch_gemm<rl::EPI_BF16, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                    group_m_for(RL_K_DH_GEMM, kGroupMBwd), e5, sms, st, 1, 0, cnt, dyn);
    }
    RL_TRY(make_map(&t_dh, out, true, H, rows, H, 32, 32));
    return launch_gemm<rl::EPI_F32, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                 group_m_for(RL_K_DH_GEMM, kGroupMBwd), e5, sms, st, 1, 0, cnt, dyn);
  }
  const int64_t rows_pad = (rows + 255) / 256 * 256;
  float* part = reinterpret_cast<float*>(ws + L.dh_split);
  CUtensorMap t_part;
  RL_TRY(make_map(&t_part, part, true, H, S * rows_pad, H, 32, 32));
  RL_TRY((launch_gemm<rl::EPI_F32, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_part, rows, H, V,
                                                group_m_for(RL_K_DH_GEMM, kGroupMBwd), e5, sms, st, S,
                                                static_cast<int>(rows_pad), cnt, dyn)));
  {
    ProfScope ps(RL_K_COMPACT, st);
    const int64_t n4 = rows * H / 4;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n4 + 255) / 256, int64_t(sms) * 8));
    if (bf16_out)
      rl::split_sum_kernel<uint16_t><<<blocks, 256, 0, st>>>(part, S, rows_pad, H, rows, cnt,
                                                             static_cast<uint16_t*>(out));
    else
      rl::split_sum_kernel<float><<<blocks, 256, 0, st>>>(part, S, rows_pad, H, rows, cnt, static_cast<float*>(out));
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

// K4 from the probability cache (forward_impl filled it in the same fused call).
rl_status launch_dz_from_cache(const rl_lm_shape* s, const uint8_t* ws, const WsLayout& L, const int32_t* row_map,
                               int64_t row0, const int* cnt, int64_t rows, const float* coef, const float* lse,
                               const int32_t* targets, const float* invt_rows, uint16_t* dz, int sms,
                               cudaStream_t st) {
  {
    ProfScope ps(RL_K_DZ_CACHE, st);
    static const int bps = [] {  // RL_DZC_BLOCKS_PER_SM: blocks per SM of the grid-stride row loop (A/B)
      const char* e = getenv("RL_DZC_BLOCKS_PER_SM");
      const int v = e ? atoi(e) : 8;
      return v > 0 ? v : 8;
    }();
    rl::dz_from_cache_kernel<<<bps * sms, rl::DZC_THREADS, 0, st>>>(
        reinterpret_cast<const uint16_t*>(ws + L.pc), reinterpret_cast<const float*>(ws + L.pm), L.ldz, s->T, row_map,
        row0, cnt, rows, s->V_local, coef, lse, targets, s->vocab_offset, invt_rows, s->inv_temperature, dz);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

// Sparse backward: the same K4 -> K6 -> K5 over the rows whose coefficient is
// non-zero only (their order kept). Row counts live on the device: the GEMMs read
// them at start (dyn_mode), so nothing synchronises the host.
rl_status bwd_sparse_impl(const rl_lm_shape* s, const uint16_t* hidden, const uint16_t* w, const int32_t* targets,
                          const float* lse, const float* coef, uint16_t* dh, float* dh32, float* dw,
                          int accumulate_dw, uint8_t* ws, const WsLayout& L, int sms, cudaStream_t st, int phases,
                          const rl_nvls_reduce* dw_nvls, const rl_nvls_reduce* dh_nvls, bool from_cache) {
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
    if ((phases & RL_BWD_DU) && from_cache) {
      RL_TRY(launch_dz_from_cache(s, ws, L, idx + c0, 0, cnt, rows, coef_c + c0, lse_c + c0, tgt_c + c0,
                                  s->inv_temperature_rows ? invt_c + c0 : nullptr, dz, sms, st));
    } else if (phases & RL_BWD_DU) {
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
      if (dw_nvls && ch == n_chunks - 1) {
        RL_TRY(launch_dw_nvls(t_dz_mn, t_h_mn, t_dw, V, H, rows, dw, dw_nvls, ch > 0 || accumulate_dw, sms, st, cnt));
      } else if (ch == 0 && !accumulate_dw) {
        RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                     group_m_for(RL_K_DW_GEMM, kGroupMBwd), e6, sms, st, 1, 0, cnt, 2)));
      } else {
        RL_TRY((launch_gemm<rl::EPI_F32_ADD, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows,
                                                         group_m_for(RL_K_DW_GEMM, kGroupMBwd), e6, sms, st, 1, 0, cnt, 2)));
      }
    }
    if ((phases & RL_BWD_DH) && (dh || dh32)) {
      RL_TRY(make_map(&t_dz_k, dz, false, V, rows, L.ldz, 64, kARows));
      rl::EpiParams e5 = {};
      e5.rows = rows;
      e5.cols = H;
      if (dh_nvls) {
        // the compact rows go straight to their own rows of the (zeroed) symmetric
        // d_hidden_f32 and are reduced there: every rank holds the same compaction
        // (S3 ran on identical inputs), so row_map is the same on all of them
        RL_TRY(make_map(&t_dh, dh_c, true, H, rows, H, 32, 32));
        set_nvls(e5, dh_nvls, dh32, 0, ch);
        e5.row_map = idx + c0;
        RL_TRY((launch_gemm<rl::EPI_F32_NVLS, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                             group_m_for(RL_K_DH_GEMM, kGroupMBwd), e5, sms, st, 1, 0,
                                                             cnt, 1)));
        continue;
      }
      RL_TRY(launch_dh(t_dz_k, t_w_mn, rows, H, V, dh_c, dh != nullptr, cnt, ws, L, sms, st));
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
                   const rl_nvls_reduce* dw_nvls = nullptr, const rl_nvls_reduce* dh_nvls = nullptr,
                   bool from_cache = false) {
  const int64_t T = s->T, H = s->H, V = s->V_local;
  if (T == 0) {
    if (dw && dw_nvls && (phases & RL_BWD_DW)) {
      // no rows on this rank: K6 with an empty K range still joins the reduction
      CUtensorMap t_any, t_dw;
      RL_TRY(make_map(&t_any, dw, false, 64, 1, 64, 64, 1));  // never loaded from
      RL_TRY(make_map(&t_dw, dw, true, H, V, H, 32, 32));
      g_sync_ctr = nullptr;
      return launch_dw_nvls(t_any, t_any, t_dw, V, H, 0, dw, dw_nvls, accumulate_dw != 0, sms, st);
    }
    if (dw && !accumulate_dw) RL_CUDA(cudaMemsetAsync(dw, 0, static_cast<size_t>(V) * H * 4, st));
    return RL_OK;
  }
  uint16_t* dz = reinterpret_cast<uint16_t*>(ws + L.dz);
  const int64_t chunk = L.chunk;
  g_sync_ctr = reinterpret_cast<uint32_t*>(ws + L.sync);
  if (!(phases & RL_BWD_DENSE))
    return bwd_sparse_impl(s, hidden, w, targets, lse, coef, dh, dh32, dw, accumulate_dw, ws, L, sms, st, phases,
                           dw_nvls, dh_nvls, from_cache);
  CUtensorMap t_h_k, t_w_k, t_dz_st, t_dz_k, t_w_mn, t_dh, t_dz_mn, t_h_mn, t_dw;
  RL_TRY(make_map(&t_w_k, w, false, H, V, H, 64, rl::BN / cta_group()));
  RL_TRY(make_map(&t_w_mn, w, false, H, V, H, 64, 64));
  if (dw) RL_TRY(make_map(&t_dw, dw, true, H, V, H, 32, 32));
  for (int64_t c0 = 0, ch = 0; c0 < T; c0 += chunk, ++ch) {
    const int64_t rows = (T - c0 < chunk) ? (T - c0) : chunk;
    const bool last = c0 + rows >= T;
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
    if ((phases & RL_BWD_DU) && from_cache)
      RL_TRY(launch_dz_from_cache(s, ws, L, nullptr, c0, nullptr, rows, coef + c0, lse + c0, targets + c0,
                                  ep.invt_rows, dz, sms, st));
    else if (phases & RL_BWD_DU)
      RL_TRY((launch_gemm<rl::EPI_DZ, false, false>(RL_K_DZ_GEMM, t_h_k, t_w_k, t_dz_st, rows, V, H, group_m_for(RL_K_DZ_GEMM, 16), ep, sms, st)));
    // K6: dW (+)= dU^T h
    if ((phases & RL_BWD_DW) && dw) {
      RL_TRY(make_map(&t_dz_mn, dz, false, V, rows, L.ldz, 64, 64));
      RL_TRY(make_map(&t_h_mn, hc, false, H, rows, H, 64, 64));
      rl::EpiParams e6 = {};
      e6.rows = V;
      e6.cols = H;
      if (dw_nvls && last) {
        RL_TRY(launch_dw_nvls(t_dz_mn, t_h_mn, t_dw, V, H, rows, dw, dw_nvls, c0 > 0 || accumulate_dw, sms, st));
      } else if (c0 == 0 && !accumulate_dw) {
        RL_TRY((launch_gemm<rl::EPI_F32, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows, group_m_for(RL_K_DW_GEMM, kGroupMBwd), e6, sms, st)));
      } else {
        RL_TRY((launch_gemm<rl::EPI_F32_ADD, true, true>(RL_K_DW_GEMM, t_dz_mn, t_h_mn, t_dw, V, H, rows, group_m_for(RL_K_DW_GEMM, kGroupMBwd), e6, sms, st)));
      }
    }
    // K5: dH chunk = dU W
    if ((phases & RL_BWD_DH) && (dh || dh32)) {
      RL_TRY(make_map(&t_dz_k, dz, false, V, rows, L.ldz, 64, kARows));
      rl::EpiParams e5 = {};
      e5.rows = rows;
      e5.cols = H;
      if (dh) {
        RL_TRY(launch_dh(t_dz_k, t_w_mn, rows, H, V, dh + c0 * H, true, nullptr, ws, L, sms, st));
      } else if (dh_nvls) {
        RL_TRY(make_map(&t_dh, dh32 + c0 * H, true, H, rows, H, 32, 32));
        set_nvls(e5, dh_nvls, dh32 + c0 * H, c0 * H, static_cast<int>(ch));
        RL_TRY((launch_gemm<rl::EPI_F32_NVLS, false, true>(RL_K_DH_GEMM, t_dz_k, t_w_mn, t_dh, rows, H, V,
                                                             group_m_for(RL_K_DH_GEMM, kGroupMBwd), e5, sms, st)));
      } else {
        RL_TRY(launch_dh(t_dz_k, t_w_mn, rows, H, V, dh32 + c0 * H, false, nullptr, ws, L, sms, st));
      }
    }
  }
  return RL_OK;
}

}  // namespace
