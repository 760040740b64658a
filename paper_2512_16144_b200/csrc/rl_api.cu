// librl host side: argument validation, workspace carving, TMA tensor maps and
// kernel launches behind the C ABI of include/rl.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <array>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/rl.h"
#include "rl_gemm.cuh"
#include "rl_small.cuh"

#include "rl_host_common.cuh"
#include "rl_launch.cuh"
#include "rl_workspace.cuh"
#include "rl_step.cuh"
#include "rl_ns_hostio.cuh"

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

int64_t rl_nvls_shard_rows(int64_t rows, int32_t world) { return nvls_shard_rows(rows, world); }

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

rl_status rl_fwd_partials_ex(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                             const int32_t* targets, float* partials, int32_t flags, void* workspace,
                             size_t workspace_bytes, void* stream) {
  g_launches = 0;
  if ((flags & ~RL_FWD_CACHE) != 0) return fail(RL_ERR_INVALID_ARGUMENT, "unknown rl_fwd_partials_ex flags %d", flags);
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
  const bool cache = (flags & RL_FWD_CACHE) != 0;
  if (cache && !L.pcache) return fail(RL_ERR_INVALID_ARGUMENT, "RL_FWD_CACHE: no probability cache (RL_P_CACHE=0)");
  const size_t need = L.dz;  // the forward's regions (the cache first, then the partials) end where dU begins
  if (shape->T > 0 && (!workspace || workspace_bytes < need))
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  DevInfo d;
  RL_TRY(device_info(d));
  return forward_impl(shape, hidden, w_vocab, targets, nullptr, nullptr, nullptr, reinterpret_cast<float4*>(partials),
                      static_cast<uint8_t*>(workspace), L, d.sms, static_cast<cudaStream_t>(stream), 0,
                      cache ? shape->T : 0);
}

rl_status rl_fwd_partials(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                          const int32_t* targets, float* partials, void* workspace, size_t workspace_bytes,
                          void* stream) {
  return rl_fwd_partials_ex(shape, hidden, w_vocab, targets, partials, 0, workspace, workspace_bytes, stream);
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

rl_status rl_rollout_stats(const rl_loss_params* params, int64_t T, int64_t V_global, const float* logprob,
                           const float* infer_logprobs, const int32_t* targets, const int32_t* rollout_offsets,
                           const uint8_t* loss_mask, float* rollout_kmin, double* rollout_logratio_sum,
                           int32_t* rollout_n_valid, void* stream) {
  g_launches = 0;
  RL_TRY(check_params(params));
  if (T < 0) return fail(RL_ERR_SHAPE, "T < 0");
  RL_NONNULL(rollout_offsets);
  RL_NONNULL(rollout_kmin);
  RL_NONNULL(rollout_logratio_sum);
  RL_NONNULL(rollout_n_valid);
  if (T > 0) {
    RL_NONNULL(logprob);
    RL_NONNULL(infer_logprobs);
  }
  DevInfo d;
  RL_TRY(device_info(d));
  const rl::LossArgs a = loss_args(params, T, V_global, logprob, infer_logprobs, targets, nullptr, rollout_offsets,
                                   loss_mask);
  {
    ProfScope ps(RL_K_LOSS, static_cast<cudaStream_t>(stream));
    rl::rollout_stats_kernel<<<params->num_rollouts, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        a, rollout_kmin, rollout_logratio_sum, rollout_n_valid);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_loss_coef_ex(const rl_loss_params* params, int64_t T, int64_t V_global, const float* logprob,
                          const float* infer_logprobs, const int32_t* targets, const float* rollout_adv,
                          const int32_t* rollout_offsets, const uint8_t* loss_mask, const float* rollout_kmin,
                          const double* rollout_logratio_sum, const int32_t* rollout_n_valid, float* coef,
                          uint8_t* token_keep, uint8_t* rollout_guarded, rl_loss_report* report, void* workspace,
                          size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_TRY(check_params(params));
  if (T < 0) return fail(RL_ERR_SHAPE, "T < 0");
  RL_NONNULL(rollout_adv);
  RL_NONNULL(rollout_offsets);
  RL_NONNULL(report);
  RL_NONNULL(rollout_kmin);
  if (params->variant == RL_LOSS_GSPO && (!rollout_logratio_sum || !rollout_n_valid))
    return fail(RL_ERR_INVALID_ARGUMENT, "GSPO over split rollouts needs rollout_logratio_sum and rollout_n_valid");
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
                   static_cast<cudaStream_t>(stream), rollout_kmin, rollout_logratio_sum, rollout_n_valid);
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
  if (dw_nvls && !d_w_vocab) return fail(RL_ERR_INVALID_ARGUMENT, "dw_nvls reduces d_w_vocab");
  if (dh_nvls && !d_hidden_f32) return fail(RL_ERR_INVALID_ARGUMENT, "dh_nvls reduces d_hidden_f32");
  if ((phases & RL_BWD_ALL) == 0 || (phases & ~(RL_BWD_ALL | RL_BWD_DENSE | RL_BWD_FROM_CACHE)) != 0)
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
  if ((phases & RL_BWD_FROM_CACHE) && !L.pcache)
    return fail(RL_ERR_INVALID_ARGUMENT, "RL_BWD_FROM_CACHE: no probability cache (RL_P_CACHE=0)");
  if ((phases & RL_BWD_ALL) != RL_BWD_ALL && L.chunk < shape->T)
    return fail(RL_ERR_INVALID_ARGUMENT, "partial backward phases need one dU chunk (dz_chunk_rows = 0 or >= T)");
  if ((dw_nvls || dh_nvls) && shape->T > 0 && (shape->T + L.chunk - 1) / L.chunk > kNvlsChunkEpochs)
    return fail(RL_ERR_INVALID_ARGUMENT, "NVLS reduction supports at most %d dU chunks", kNvlsChunkEpochs);
  DevInfo d;
  RL_TRY(device_info(d));
  int sms = d.sms;
  if (max_sms > 0 && max_sms < sms) sms = max_sms < 2 ? 2 : max_sms;
  return bwd_impl(shape, hidden, w_vocab, targets, lse, coef, d_hidden, d_hidden_f32, d_w_vocab, accumulate_dw,
                  static_cast<uint8_t*>(workspace), L, sms, static_cast<cudaStream_t>(stream),
                  phases & ~RL_BWD_FROM_CACHE, dw_nvls, dh_nvls, (phases & RL_BWD_FROM_CACHE) != 0);
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
                          out->entropy ? out->entropy + r0 : nullptr, lse + r0, nullptr, ws, L, sms, st, r0,
                          shape->T));
    }
  } else {
    RL_TRY(forward_impl(shape, hidden, w_vocab, targets, out->logprob, out->entropy, lse, nullptr, ws, L, sms, st, 0,
                        shape->T));
  }
  RL_TRY(loss_impl(params, shape->T, shape->V_global, out->logprob, infer_logprobs, targets, rollout_adv,
                   rollout_offsets, loss_mask, coef, out->token_keep, out->rollout_guarded, out->report,
                   reinterpret_cast<rl::RolloutPartial*>(ws + L.rp), st));
  RL_TRY(bwd_impl(shape, hidden, w_vocab, targets, lse, coef, out->d_hidden, out->d_hidden_f32, out->d_w_vocab,
                  out->accumulate_dw, ws, L, sms, st, RL_BWD_ALL | (out->dense_backward ? RL_BWD_DENSE : 0),
                  out->d_w_vocab_nvls, nullptr, L.pcache));
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
  if (out->d_w_vocab_nvls && !out->d_w_vocab)
    return fail(RL_ERR_INVALID_ARGUMENT, "d_w_vocab_nvls reduces d_w_vocab");
  if (out->dz_chunk_rows < 0) return fail(RL_ERR_INVALID_ARGUMENT, "dz_chunk_rows must be >= 0");
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
  HostioStreams* hsp = nullptr;
  RL_TRY(hostio_streams(hsp));
  HostioStreams& hs = *hsp;
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

rl_status rl_fold_gamma(const uint16_t* w, const float* gamma, int64_t rows, int64_t K, uint16_t* out,
                        void* stream) {
  g_launches = 0;
  if (rows < 0 || K < 8 || K % 8) return fail(RL_ERR_SHAPE, "need rows >= 0 and K a positive multiple of 8");
  if (rows == 0) return RL_OK;
  RL_NONNULL(w);
  RL_NONNULL(gamma);
  RL_NONNULL(out);
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(out)) & 15 ||
      reinterpret_cast<uintptr_t>(gamma) & 15)
    return fail(RL_ERR_INVALID_ARGUMENT, "w, gamma and out must be 16-byte aligned");
  DevInfo d;
  RL_TRY(device_info(d));
  const int64_t n8 = rows * K / 8;
  const int64_t blocks = std::min<int64_t>((n8 + 255) / 256, static_cast<int64_t>(d.sms) * 8);
  {
    ProfScope ps(RL_K_NS_AUX, static_cast<cudaStream_t>(stream));
    rl::fold_gamma_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        w, gamma, rows, K, out);
  }
  RL_CHECK_LAUNCH();
  return RL_OK;
}

rl_status rl_expert_load(const int32_t* offsets, int32_t n_groups, int64_t rows, float* out, void* stream) {
  g_launches = 0;
  if (n_groups < 1 || rows < 0) return fail(RL_ERR_SHAPE, "need n_groups >= 1 and rows >= 0");
  RL_NONNULL(offsets);
  RL_NONNULL(out);
  {
    ProfScope ps(RL_K_NS_AUX, static_cast<cudaStream_t>(stream));
    rl::expert_load_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(offsets, n_groups, rows, out);
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

static rl_status ns_shard_check(int64_t M, int64_t N, int32_t steps, void* workspace, size_t workspace_bytes,
                                NsLayout& l, DevInfo& d) {
  RL_TRY(check_ns_shape(M, N, steps));
  if (M < N) return fail(RL_ERR_SHAPE, "row-sharded Newton-Schulz needs M_local >= N (tall shards)");
  if (!aligned16(workspace)) return fail(RL_ERR_ALIGNMENT, "workspace must be 16-byte aligned");
  l = ns_layout(M, N, false);
  if (!workspace || workspace_bytes < l.end)
    return fail(RL_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", l.end, workspace_bytes);
  return device_info(d);
}

rl_status rl_ns_shard_sumsq(const float* g, int64_t M_local, int64_t N, double* sumsq, void* workspace,
                            size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_NONNULL(g);
  RL_NONNULL(sumsq);
  if (!aligned16(g)) return fail(RL_ERR_ALIGNMENT, "g must be 16-byte aligned");
  NsLayout l;
  DevInfo d;
  RL_TRY(ns_shard_check(M_local, N, 1, workspace, workspace_bytes, l, d));
  return ns_shard_sumsq_impl(g, M_local, N, sumsq, static_cast<uint8_t*>(workspace), l,
                             static_cast<cudaStream_t>(stream));
}

rl_status rl_ns_shard_gram(int32_t j, const float* g, const double* sumsq, int64_t M_local, int64_t N, float* gram,
                           void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_NONNULL(gram);
  if (j < 0) return fail(RL_ERR_INVALID_ARGUMENT, "iteration j must be >= 0");
  if (j == 0) {
    RL_NONNULL(g);
    RL_NONNULL(sumsq);
    if (!aligned16(g)) return fail(RL_ERR_ALIGNMENT, "g must be 16-byte aligned");
  }
  if (!aligned16(gram)) return fail(RL_ERR_ALIGNMENT, "gram must be 16-byte aligned");
  NsLayout l;
  DevInfo d;
  RL_TRY(ns_shard_check(M_local, N, 1, workspace, workspace_bytes, l, d));
  return ns_shard_gram_impl(j, g, sumsq, M_local, N, gram, static_cast<uint8_t*>(workspace), l, d.sms,
                            static_cast<cudaStream_t>(stream));
}

rl_status rl_ns_shard_apply(int32_t j, int32_t steps, const float* gram, int64_t M_local, int64_t N, uint16_t* out,
                            void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  RL_NONNULL(gram);
  if (j < 0 || j >= steps) return fail(RL_ERR_INVALID_ARGUMENT, "need 0 <= j < steps");
  if (j == steps - 1) {
    RL_NONNULL(out);
    if (!aligned16(out)) return fail(RL_ERR_ALIGNMENT, "out must be 16-byte aligned");
  }
  NsLayout l;
  DevInfo d;
  RL_TRY(ns_shard_check(M_local, N, steps, workspace, workspace_bytes, l, d));
  return ns_shard_apply_impl(j, steps, gram, M_local, N, out, static_cast<uint8_t*>(workspace), l, d.sms,
                             static_cast<cudaStream_t>(stream));
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

#ifdef RL_AB_STATS
// A/B build only (not in include/rl.h): copy the per-CTA cycle counters of the last launch
// of epilogue mode `mode` (rl_gemm.cuh, g_ab_stats) to host memory `out` [512][8].
extern "C" int32_t rl_ab_stats_read(int32_t mode, unsigned long long* out) {
  if (mode < 0 || mode >= 8) return -1;
  if (cudaMemcpyFromSymbol(out, rl::g_ab_stats, sizeof(unsigned long long) * 512 * 8,
                           sizeof(unsigned long long) * 512 * 8 * mode) != cudaSuccess)
    return -2;
  return 0;
}
#endif
