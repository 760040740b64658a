/*
 * librl — B200-native fused LM-head + IcePop policy-loss step (C ABI).
 *
 * The operation is the per-token policy-gradient loss of PAPER.md §3.3
 * (arXiv 2512.16144, INTELLECT-3), lines 449-472:
 *
 *   Eq.1 (L451-463)  J = 1/sum_i|y_i| * sum_i sum_t M(pi_train(y_it)/pi_infer(y_it); a, b) * A_it
 *   Eq.2 (L465-468)  M(k) = k if k in [a, b] else 0          (a = 0.5, b = 5 by default)
 *   L470             A_it = S_i - mean_G(S)                   (no std division)
 *   L472             a rollout is masked if any of its token ratios < 1e-5
 *
 * where log pi_train(y_t) is the log-softmax, at the sampled token, of the LM
 * head logits z_t = invT * W_vocab h_t over the full vocabulary. The library
 * minimises loss = -J and returns d loss / d hidden and d loss / d W_vocab.
 * The readings of every point the paper leaves open are listed in DESIGN.md §2
 * (R1-R20) and cited below as "R<n>". Options beyond Eq.1 (loss variants R16/R17,
 * the KL term R19, per-token temperature R20) are off by default.
 *
 * Conventions for every call:
 *  - Pointers are DEVICE pointers unless the argument says HOST. The caller
 *    owns and allocates every buffer, including the workspace; the library
 *    never allocates device memory, never frees, and never synchronises the
 *    device (the *_hostio call is the one exception: it waits on `stream`).
 *  - bf16 tensors are passed as uint16_t bit patterns. All matrices are
 *    row-major and contiguous along the hidden dimension: hidden [T, H],
 *    W_vocab [V_local, H] (the nn.Linear layout, no transpose), d_hidden [T, H],
 *    d_w_vocab [V_local, H].
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - Host-checkable errors (null pointers, bad sizes, misaligned pointers,
 *    bad parameters, short workspace, a device that is not sm_100) return a
 *    status synchronously with a message from rl_last_error_message(), and
 *    enqueue nothing. Data-dependent problems (non-finite or positive stored
 *    log-probs, targets outside [0, V_global), malformed rollout offsets) are
 *    counted in rl_loss_report and neutralised on the device (R-faults in
 *    DESIGN.md §4): the token is excluded, or, for bad offsets, the whole batch
 *    gets coef = 0.
 *  - Every 16-byte-vectorised pointer (hidden, W_vocab, d_hidden, d_w_vocab,
 *    workspace) must be 16-byte aligned; H must be a multiple of 8.
 *  - A workspace belongs to one call at a time: calls that may execute
 *    concurrently (different streams) need different workspaces (the GEMMs keep
 *    their soft k-barrier counters there; rl_bwd_ex phases also keep dU there).
 */
#ifndef RL_H_
#define RL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RL_ABI_VERSION 3

typedef enum rl_status {
  RL_OK = 0,
  RL_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad parameter value           */
  RL_ERR_SHAPE = 2,            /* size out of range or inconsistent          */
  RL_ERR_UNSUPPORTED = 3,      /* device is not sm_100, or feature not built  */
  RL_ERR_CUDA = 4,             /* a CUDA runtime/driver call failed          */
  RL_ERR_WORKSPACE = 5,        /* workspace null or smaller than required    */
  RL_ERR_ALIGNMENT = 6         /* pointer not 16-byte aligned                */
} rl_status;

/* Shape of the LM-head contraction on this rank. */
typedef struct rl_lm_shape {
  int64_t T;               /* packed token rows (>= 0)                              */
  int64_t H;               /* hidden size (multiple of 8, <= 65536)                  */
  int64_t V_local;         /* rows of W_vocab on this rank (>= 1)                    */
  int64_t vocab_offset;    /* global id of W_vocab row 0 (vocab-parallel shard start) */
  int64_t V_global;        /* full vocabulary size (>= vocab_offset + V_local)       */
  float inv_temperature;   /* 1/tau applied to the logits, > 0 (R8; default 1)       */
  int32_t _pad;
  const float* inv_temperature_rows; /* optional DEVICE [T] per-token 1/tau (> 0, finite;
                              reading R20), overriding inv_temperature; NULL = scalar.
                              Row t of every call's T rows (vocab shards share it).     */
} rl_lm_shape;

/* Loss variants. All share the backward: each only changes
 * coef_t = -d loss / d logp_t and the loss value (R16, R17).
 *   RL_LOSS_ICEPOP  Eq.1 + Eq.2: token ratio masked outside [alpha, beta] (the paper)
 *   RL_LOSS_CISPO   ratio clipped to [alpha, beta], as a stop-gradient weight on
 *                   log pi (CISPO, contrasted with IcePop at PAPER.md L472)
 *   RL_LOSS_GSPO    sequence-level ratio s_i = exp(mean_t log k_t), PPO-style clip of s_i
 *                   to [alpha, beta] (GSPO, Fig. 8); D is then the
 *                   caller's sequence count */
typedef enum rl_loss_variant { RL_LOSS_ICEPOP = 0, RL_LOSS_CISPO = 1, RL_LOSS_GSPO = 2 } rl_loss_variant;

/* Loss hyper-parameters. */
typedef struct rl_loss_params {
  float alpha;             /* Eq.2 lower bound, 0 < alpha <= 1 (clip low for CISPO/GSPO) */
  float beta;              /* Eq.2 upper bound, beta >= 1, closed interval (R4)           */
  float guard_threshold;   /* rollout masked iff min_t k_t < guard (strict, R4); 0 off    */
  int32_t num_rollouts;    /* R = number of packed rollouts on this rank (>= 1)          */
  double loss_denominator; /* D = sum_i |y_i| over the GLOBAL step batch, > 0 (R5)        */
  int32_t variant;         /* rl_loss_variant; 0 = the paper's IcePop objective           */
  int32_t kl_set;          /* rl_kl_set: the tokens the KL term covers                    */
  float kl_tau;            /* KL term weight (reading R19): loss += (kl_tau/D) sum_{t in S}
                              log k_t, coef_t -= kl_tau/D on S; 0 = off (the paper)         */
  int32_t _pad;
} rl_loss_params;

/* Token set S of the KL term (reading R19): Eq.2/guard-masked valid tokens, kept
 * tokens, or every valid loss token. */
typedef enum rl_kl_set { RL_KL_MASKED = 0, RL_KL_UNMASKED = 1, RL_KL_ALL = 2 } rl_kl_set;

/* Device-resident loss report (SPEC LossReport + counters). Written, not
 * accumulated, by every call that takes it. Sums use a fixed-order reduction,
 * so two identical calls give bit-identical reports. */
typedef struct rl_loss_report {
  double loss;               /* -J contribution of this rank: -(1/D) sum_t coef_t*D (R3) */
  double mismatch_kl_sum;    /* sum over valid tokens of k - log k - 1                  */
  uint32_t kept_tokens;      /* tokens with keep = 1                                    */
  uint32_t masked_low;       /* valid tokens with k < alpha                             */
  uint32_t masked_high;      /* valid tokens with k > beta                              */
  uint32_t guarded_rollouts; /* rollouts with min k < guard                             */
  uint32_t guarded_tokens;   /* valid tokens inside guarded rollouts                    */
  uint32_t nonfinite_inputs; /* loss tokens whose stored log-prob is NaN/inf or > 0     */
  uint32_t bad_targets;      /* loss tokens whose target is outside [0, V_global)       */
  uint32_t bad_offsets;      /* 1 if rollout_offsets is not 0 = o_0 <= ... <= o_R = T  */
} rl_loss_report;

/* Fused cross-rank reduction of an fp32 output over an NVLink multicast group
 * (NVLS), done inside the producing GEMM's epilogue: every rank stores its own
 * contribution into its replica of a symmetric buffer (the usual output pointer),
 * publishes a per-slab flag (32 output rows), and the slab's owner sums it over
 * all replicas with multimem.ld_reduce.
 *   mode RL_NVLS_ALL_REDUCE (0): the owner is tile % world and writes the sum to
 *     every replica with multimem.st; after the call, and after a cross-rank
 *     barrier the caller runs on the same stream, every replica holds the sum.
 *   mode RL_NVLS_REDUCE_SCATTER (1, FSDP-consistent): rank r owns the
 *     output rows [r S, min((r+1) S, rows)), S = rl_nvls_shard_rows(rows, world),
 *     and writes their sum to its own replica only (half the NVLink traffic);
 *     its other rows keep its own contribution.
 * Requirements: the output pointer is this rank's view of the symmetric buffer
 * whose multicast VA is `multicast`; each flag array holds rl_nvls_flag_count()
 * uint32 entries, zeroed once at allocation; `epoch` increases on every call
 * (0 < epoch < 2^24; a flag holds epoch * 256 + dU chunk, so a call may run up to
 * 256 dU chunks); all ranks make the same call with the same shapes. A rank with
 * T = 0 still takes part (its dW GEMM runs with an empty K range), so DP ranks may
 * hold different row counts.
 * Accumulation (d_w_vocab): with accumulate_dw = 1 the rank's new gradient is
 * added to what its replica already holds (earlier micro-batches, each run with
 * accumulate_dw and no descriptor) and the SUM is reduced, once, in the dW GEMM of
 * the last dU chunk: the deferred reduction of a gradient-accumulation step.
 * Sparse backward (d_hidden_f32, vocab-parallel): the compacted rows are stored
 * straight into their own rows of the replica, which is zeroed first, and reduced
 * there; every rank must hold the same coefficients (S3 on identical inputs). */
#define RL_NVLS_MAX_RANKS 8
typedef struct rl_nvls_reduce {
  void* multicast;                    /* multicast VA of the symmetric fp32 output buffer  */
  uint32_t* flags[RL_NVLS_MAX_RANKS]; /* every rank's flag array (peer VAs); [rank] = local */
  int32_t rank;                       /* this rank in the multicast group                  */
  int32_t world;                      /* ranks in the group, 2..RL_NVLS_MAX_RANKS          */
  uint32_t epoch;                     /* > every epoch used before with these flags        */
  int32_t lag;                        /* 0: dedicated warps reduce each slab as soon as every
                                         rank published it (default); > 0: the epilogue warps
                                         reduce the slab stored `lag` tiles earlier (A/B)     */
  int32_t mode;                       /* rl_nvls_mode                                      */
  int32_t _pad;
} rl_nvls_reduce;
typedef enum rl_nvls_mode { RL_NVLS_ALL_REDUCE = 0, RL_NVLS_REDUCE_SCATTER = 1 } rl_nvls_mode;

/* Rows per rank of the reduce-scatter mode: ceil(rows / (32 world)) * 32 (whole slabs). */
int64_t rl_nvls_shard_rows(int64_t rows, int32_t world);

/* Outputs of rl_policy_loss_fwd_bwd. Optional pointers may be NULL. */
typedef struct rl_loss_outputs {
  rl_loss_report* report;  /* [1] device, required                                     */
  float* logprob;          /* [T] log pi_train(y_t), required                          */
  float* entropy;          /* [T] entropy of the scaled distribution (R9), optional    */
  float* lse;              /* [T] log-sum-exp of the scaled logits, optional           */
  float* coef;             /* [T] keep_t k_t A_i / D (d loss / d logp_t = -coef_t), opt */
  uint8_t* token_keep;     /* [T] 1 if the token contributes, optional                 */
  uint8_t* rollout_guarded;/* [R] 1 if the rollout was masked by the guard, optional   */
  uint16_t* d_hidden;      /* [T, H] bf16 d loss / d hidden; or NULL                    */
  float* d_hidden_f32;     /* [T, H] fp32 alternative (vocab-parallel partial); or NULL */
  float* d_w_vocab;        /* [V_local, H] fp32 d loss / d W_vocab; or NULL             */
  int32_t accumulate_dw;   /* 0: d_w_vocab is overwritten; 1: the gradient is added     */
  int32_t dense_backward;  /* 0 (default): the backward GEMMs run over the rows with a
                              non-zero coef only (RL_BWD_DENSE); 1: over all T rows     */
  const rl_nvls_reduce* d_w_vocab_nvls; /* non-NULL: d_w_vocab is all-reduced in the dW
                             GEMM epilogue of the last dU chunk over NVLS (data-parallel
                             ranks); with accumulate_dw = 1 the sum of the replica's old
                             contents and this step's gradient is reduced                */
  int64_t dz_chunk_rows;   /* rows of the bf16 dU buffer per backward pass; 0 = T (size
                              the workspace with the same value)                         */
} rl_loss_outputs;

/* ---------------------------------------------------------------- S0 */
/* A[g*G + j] = rewards[g*G + j] - mean_j rewards[g*G + j].
 * rewards, advantages: [num_groups * group_size] fp32, group-major.
 * group_size < 2 -> RL_ERR_INVALID_ARGUMENT (no baseline). */
rl_status rl_group_advantages(const float* rewards, int32_t num_groups, int32_t group_size,
                              float* advantages, void* stream);

/* ------------------------------------------------------------- S1 + S2 */
/* logprob[t] = z_t[y_t] - lse_t,  entropy[t] = -sum_v p_tv log p_tv,  lse[t],
 * with z_t = invT * W h_t over the full vocabulary (Eq.1's pi_train). The
 * logits exist only in tensor memory; nothing T x V touches HBM.
 * Requires V_local == V_global (single shard); vocab-parallel callers use
 * rl_fwd_partials + rl_merge_partials. entropy and lse may be NULL. */
rl_status rl_logprob_fwd(const rl_lm_shape* shape, const uint16_t* hidden,
                         const uint16_t* w_vocab, const int32_t* targets, float* logprob,
                         float* entropy, float* lse, void* workspace, size_t workspace_bytes,
                         void* stream);

/* ----------------------------------------------------------- S0 .. S6 */
/* The whole step for one rank: logits (TMEM only) -> online log-softmax ->
 * k_t = exp(logprob_t - infer_logprobs_t) -> Eq.2 gate + rollout guard ->
 * coef_t -> loss, then the backward d loss / d u_tv = coef_t invT (p_tv - [v==y_t])
 * folded into d_hidden = dU W and d_w_vocab = dU^T hidden. By default the
 * backward GEMMs run over the rows with coef_t != 0 only (their dU row is the
 * only non-zero one); d_hidden rows of the others are written as zeros.
 *   targets          [T] int32 global vocab ids (row t is scored on targets[t];
 *                    shifting labels is the caller's job)
 *   infer_logprobs   [T] fp32, log pi_infer(y_t) as stored by the inference engine
 *   rollout_adv      [R] fp32, A_i (from rl_group_advantages)
 *   rollout_offsets  [R+1] int32 CSR row offsets of the packed rollouts
 *   loss_mask        [T] uint8 or NULL (= all ones); 0 rows get logprob/entropy
 *                    but no loss, guard participation or gradient (R4, R5)
 * Requires V_local == V_global; vocab-parallel callers use the split phases. */
rl_status rl_policy_loss_fwd_bwd(const rl_lm_shape* shape, const rl_loss_params* params,
                                 const uint16_t* hidden, const uint16_t* w_vocab,
                                 const int32_t* targets, const float* infer_logprobs,
                                 const float* rollout_adv, const int32_t* rollout_offsets,
                                 const uint8_t* loss_mask, const rl_loss_outputs* out,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* Same step with the per-step inputs in HOST memory (pinned for async copies):
 * hidden_host, targets_host, infer_host, rewards_host ([R] fp32, grouped by
 * group_size), offsets_host, loss_mask_host (or NULL) are copied into the
 * workspace on `stream`, advantages are computed on the device, the step runs,
 * and the report is copied back to report_host before returning (the call
 * synchronises `stream`). W_vocab, d_hidden and d_w_vocab stay on the device
 * (they are model state). Workspace: rl_workspace_bytes_hostio. */
rl_status rl_policy_loss_fwd_bwd_hostio(const rl_lm_shape* shape, const rl_loss_params* params,
                                        int32_t group_size, const uint16_t* hidden_host,
                                        const uint16_t* w_vocab, const int32_t* targets_host,
                                        const float* infer_host, const float* rewards_host,
                                        const int32_t* offsets_host, const uint8_t* loss_mask_host,
                                        const rl_loss_outputs* out, rl_loss_report* report_host,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------- split phases (vocab-parallel) */
/* S1 on the local shard, reduced to ONE partial per row:
 * partials[t] = (m_t, s_t, u_t, zt_t) with, over the shard's scaled logits,
 * m = max z, s = sum e^{z-m}, u = sum e^{z-m}(z-m), zt = z_{y_t} if y_t is in
 * [vocab_offset, vocab_offset + V_local) else -inf.  partials: [T] float4 (16 B/row). */
rl_status rl_fwd_partials(const rl_lm_shape* shape, const uint16_t* hidden,
                          const uint16_t* w_vocab, const int32_t* targets, float* partials,
                          void* workspace, size_t workspace_bytes, void* stream);
/* rl_fwd_partials with flags: RL_FWD_CACHE also stores the probability cache (fp16 softmax
 * numerators of this shard and per-32-column maxima) into the workspace for a later
 * rl_bwd_ex(phases | RL_BWD_FROM_CACHE) with the same inputs and workspace (a workspace of
 * rl_workspace_bytes(shape, ...) holds it; RL_ERR_WORKSPACE if it is too small). */
#define RL_FWD_CACHE 1
rl_status rl_fwd_partials_ex(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                             const int32_t* targets, float* partials, int32_t flags, void* workspace,
                             size_t workspace_bytes, void* stream);

/* S2: merge n_parts partial arrays ([n_parts, T] float4, e.g. all-gathered from
 * every vocab shard, merged in index order) into logprob, entropy, lse ([T]). */
rl_status rl_merge_partials(const float* partials, int32_t n_parts, int64_t T, float* logprob,
                            float* entropy, float* lse, void* stream);

/* S3: Eq.1/Eq.2/guard (or the params' variant, plus the optional KL term R19)
 * from logprob. Writes coef [T] (required; d loss / d logprob_t = -coef_t),
 * token_keep, rollout_guarded (optional) and the report. targets/V_global only
 * feed the bad-target counter (targets may be NULL to skip it). */
rl_status rl_loss_coef(const rl_loss_params* params, int64_t T, int64_t V_global,
                       const float* logprob, const float* infer_logprobs, const int32_t* targets,
                       const float* rollout_adv, const int32_t* rollout_offsets,
                       const uint8_t* loss_mask, float* coef, uint8_t* token_keep,
                       uint8_t* rollout_guarded, rl_loss_report* report, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Rollouts split across ranks (packed rows sharded by sequence, so a
 * rollout's tokens may sit on several ranks). The guard of PAPER.md L472 (min over the
 * rollout's tokens) and GSPO's sequence ratio (R17) then need the whole rollout:
 *   1. rl_rollout_stats: per local rollout i (rows [offsets[i], offsets[i+1]) of this
 *      rank), over its valid loss tokens: rollout_kmin[i] = min k
 *      (+inf if none), rollout_logratio_sum[i] = sum log k (fp64), rollout_n_valid[i].
 *   2. the caller reduces them over the ranks that hold parts of the same rollout:
 *      all-reduce MIN of kmin, SUM of logratio_sum and n_valid (R floats each).
 *   3. rl_loss_coef_ex: rl_loss_coef with those reduced statistics in place of the local
 *      ones (logratio_sum / n_valid may be NULL except for GSPO). A GSPO rollout adds
 *      n_local / n_valid of its sequence term to this rank's loss, so the ranks' losses
 *      sum to the whole batch's. report.guarded_rollouts counts the guarded rollouts with
 *      rows on this rank (a split rollout is counted by every rank that holds part of it);
 *      every token counter is exact per rank.
 * rollout_adv holds the advantages of the local rollouts (from the whole groups' rewards);
 * rollout_offsets are local (0 .. T). Arrays are DEVICE [num_rollouts]. */
rl_status rl_rollout_stats(const rl_loss_params* params, int64_t T, int64_t V_global, const float* logprob,
                           const float* infer_logprobs, const int32_t* targets, const int32_t* rollout_offsets,
                           const uint8_t* loss_mask, float* rollout_kmin, double* rollout_logratio_sum,
                           int32_t* rollout_n_valid, void* stream);
rl_status rl_loss_coef_ex(const rl_loss_params* params, int64_t T, int64_t V_global, const float* logprob,
                          const float* infer_logprobs, const int32_t* targets, const float* rollout_adv,
                          const int32_t* rollout_offsets, const uint8_t* loss_mask, const float* rollout_kmin,
                          const double* rollout_logratio_sum, const int32_t* rollout_n_valid, float* coef,
                          uint8_t* token_keep, uint8_t* rollout_guarded, rl_loss_report* report, void* workspace,
                          size_t workspace_bytes, void* stream);

/* S4-S6 on the local shard, given lse and coef for every row:
 * dU = coef invT (softmax - onehot) recomputed chunk by chunk (dz_chunk_rows
 * rows at a time, 0 = all T), d_hidden(_f32) = dU W_shard (a partial sum over
 * the shard when vocab-parallel), d_w_vocab (+)= dU^T hidden. */
rl_status rl_bwd(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                 const int32_t* targets, const float* lse, const float* coef, uint16_t* d_hidden,
                 float* d_hidden_f32, float* d_w_vocab, int32_t accumulate_dw,
                 int64_t dz_chunk_rows, void* workspace, size_t workspace_bytes, void* stream);

/* rl_bwd with a phase selection and an SM budget:
 *   phases  = OR of RL_BWD_DU (K4: recompute dU into the workspace), RL_BWD_DW
 *             (K6: d_w_vocab) and RL_BWD_DH (K5: d_hidden); they run in the order
 *             DU, DW, DH. Calling DW and/or DH without DU reuses the dU left in the
 *             workspace by an earlier call with the same arguments; that requires a
 *             single dU chunk (dz_chunk_rows = 0 or >= T), else INVALID_ARGUMENT.
 *   max_sms = 0 for the whole GPU, else the persistent GEMM grids use at most
 *             this many SMs (leaving the rest to a concurrent collective).
 *   dw_nvls / dh_nvls = NULL, or all-reduce d_w_vocab / d_hidden_f32 over an NVLS
 *             group inside the K6 / K5 epilogue (see rl_nvls_reduce: dW once, in the
 *             last dU chunk; dH chunk by chunk, dense or sparse). */
#define RL_BWD_DU 1
#define RL_BWD_DW 2
#define RL_BWD_DH 4
#define RL_BWD_ALL 7
/* By default the backward runs only over the rows whose coefficient is non-zero
 * (tokens masked by Eq.2, guarded rollouts, loss_mask = 0 rows have an all-zero dU
 * row): K3's coef is compacted on the device (order kept), the hidden rows are
 * gathered, and d_hidden rows of skipped tokens are written as zeros. OR
 * RL_BWD_DENSE into `phases` to run over every row (bitwise-reproducible either
 * way; the two differ only in fp32 summation order of dW). */
#define RL_BWD_DENSE 8
/* OR into `phases`: K4 reads the probability cache that rl_fwd_partials_ex(RL_FWD_CACHE) wrote into this
 * workspace for the same shape, hidden, w_vocab and targets, instead of recomputing the logits
 * (RL_ERR_INVALID_ARGUMENT if the workspace layout has no cache, i.e. RL_P_CACHE=0). */
#define RL_BWD_FROM_CACHE 16
rl_status rl_bwd_ex(const rl_lm_shape* shape, const uint16_t* hidden, const uint16_t* w_vocab,
                    const int32_t* targets, const float* lse, const float* coef, uint16_t* d_hidden,
                    float* d_hidden_f32, float* d_w_vocab, int32_t accumulate_dw, int64_t dz_chunk_rows,
                    int32_t phases, int32_t max_sms, const rl_nvls_reduce* dw_nvls,
                    const rl_nvls_reduce* dh_nvls, void* workspace, size_t workspace_bytes, void* stream);

/* Flag entries an rl_nvls_reduce needs for d_w_vocab (which = 0) or for
 * d_hidden_f32 (which = 1) of this shape. */
int64_t rl_nvls_flag_count(const rl_lm_shape* shape, int32_t which);

/* ------------------------------------------ Muon */
/* Newton-Schulz orthogonalisation of an fp32 matrix G [M, N] (row-major, e.g.
 * d_w_vocab), the step Muon applies to a gradient (§2.1.7;
 * reading R18): X_0 = bf16(G / (||G||_F + 1e-7)), then `steps` quintic iterations
 * (a, b, c) = (3.4445, -4.7750, 2.0315):
 *   M >= N:  A = X^T X,  X <- X (a I + b A + c A^2)
 *   M <  N:  A = X X^T,  X <- (a I + b A + c A^2) X
 * Every product runs on the tcgen05 GEMMs (bf16 operands, fp32 accumulation).
 * out: [M, N] bf16. M, N >= 1, N % 8 == 0, min(M, N) % 8 == 0, steps >= 1. */
rl_status rl_newton_schulz(const float* g, int64_t M, int64_t N, int32_t steps, uint16_t* out, void* workspace,
                           size_t workspace_bytes, void* stream);
size_t rl_newton_schulz_workspace_bytes(int64_t M, int64_t N);

/* The same Newton-Schulz with G row-sharded across ranks (tall: the rows of
 * d_w_vocab, e.g. after the NVLS reduce-scatter; P:L179-181 distributed Muon).
 * X^T X = sum over ranks of X_r^T X_r, so the ranks only exchange an N x N Gram
 * per iteration and one scalar; each rank updates its own rows (X_r <- X_r C).
 * The caller runs, with G_r [M_local, N] fp32 and the same workspace throughout:
 *   rl_ns_shard_sumsq(G_r -> sumsq[1] fp64)          then all-reduce(sumsq, SUM)
 *   for j in 0..steps-1:
 *     rl_ns_shard_gram(j, G_r, sumsq -> gram [N, N] fp32)  then all-reduce(gram, SUM)
 *     rl_ns_shard_apply(j, steps, gram -> out_r [M_local, N] bf16 on the last j)
 * (j = 0 also forms X_0 = bf16(G_r / (sqrt(sumsq) + 1e-7))). Requires M_local >= N;
 * workspace: rl_newton_schulz_workspace_bytes(M_local, N). */
rl_status rl_ns_shard_sumsq(const float* g, int64_t M_local, int64_t N, double* sumsq, void* workspace,
                            size_t workspace_bytes, void* stream);
rl_status rl_ns_shard_gram(int32_t j, const float* g, const double* sumsq, int64_t M_local, int64_t N,
                           float* gram, void* workspace, size_t workspace_bytes, void* stream);
rl_status rl_ns_shard_apply(int32_t j, int32_t steps, const float* gram, int64_t M_local, int64_t N,
                            uint16_t* out, void* workspace, size_t workspace_bytes, void* stream);

/* One Muon update of an fp32 parameter matrix theta [M, N] (reading R18):
 *   m <- mu m + g;  u = nesterov ? g + mu m : m;
 *   theta <- theta (1 - lr wd) - lr sqrt(max(1, M/N)) NS_steps(u).
 * momentum [M, N] fp32 is updated in place. Workspace: rl_muon_workspace_bytes. */
rl_status rl_muon_step(float* theta, const float* grad, float* momentum, int64_t M, int64_t N, float lr, float mu,
                       float weight_decay, int32_t nesterov, int32_t steps, void* workspace, size_t workspace_bytes,
                       void* stream);
size_t rl_muon_workspace_bytes(int64_t M, int64_t N);

/* -------------------------------- MoE grouped GEMM */
/* out[r, :] = a[r, :] . b[g]^T for every row r of group g = [offsets[g], offsets[g+1]):
 * the torch._grouped_mm that PAPER.md Fig. 5 times for the MoE expert projections
 * (§2.1.8; hidden 4096, MoE dim 1408 at the GLM-4.5-Air shape).
 *   a: [rows, K] bf16 (tokens permuted so each expert's rows are contiguous)
 *   b: [n_groups, N, K] bf16 (each expert's nn.Linear weight, no transpose)
 *   offsets: [n_groups + 1] int32, DEVICE, non-decreasing, 0 .. rows (values are
 *            clamped to that range on the device; they are not otherwise validated)
 *   row_scale: NULL or [rows] fp32: out[r, :] = row_scale[r] * (a[r, :] . b[g]^T), applied
 *            to the fp32 accumulator. With row_scale = rl_rms_inv(a) and b = W o gamma
 *            (the RMSNorm weight folded into the expert weights along K) this is the
 *            expert GEMM of RMSNorm(x): diag(1/rms(x)) x (W o gamma)^T.
 *   out: [rows, N] bf16.  K % 8 == 0, N % 32 == 0, 1 <= n_groups <= 1024. */
rl_status rl_grouped_gemm(const uint16_t* a, const uint16_t* b, const int32_t* offsets, int32_t n_groups,
                          int64_t rows, int64_t N, int64_t K, const float* row_scale, uint16_t* out, void* stream);

/* out[r] = 1 / sqrt(mean_k x[r, k]^2 + eps) for bf16 x [rows, K] (the RMSNorm scale). */
rl_status rl_rms_inv(const uint16_t* x, int64_t rows, int64_t K, float eps, float* out, void* stream);

/* RMSNorm weight folded into the expert weights along K (the pre-MoE
 * norm of PAPER.md §2.1.8): out[r, k] = bf16_rn(w[r, k] * gamma[k]) for bf16 w [rows, K]
 * (all experts' weights stacked, rows = n_groups * N) and fp32 gamma [K]. Run once per
 * optimizer step; then rl_grouped_gemm(a, out, offsets, row_scale = rl_rms_inv(a)) is the
 * expert GEMM of RMSNorm(a). out may alias w. K % 8 == 0; w, gamma, out 16-byte aligned
 * (RL_ERR_INVALID_ARGUMENT otherwise). HBM-bound: 4 B per element moved. */
rl_status rl_fold_gamma(const uint16_t* w, const float* gamma, int64_t rows, int64_t K, uint16_t* out,
                        void* stream);

/* Expert load balance from the DEVICE group offsets of rl_grouped_gemm:
 * out[0] = max_g load_g, out[1] = mean load, out[2] = MaxViolation = (max - mean) / mean
 * (0 when no row is routed). load_g = the group's row count after the same clamping
 * rl_grouped_gemm applies. out: 3 fp32 on the device. */
rl_status rl_expert_load(const int32_t* offsets, int32_t n_groups, int64_t rows, float* out, void* stream);

/* ------------------------------------------------------------ utilities */
/* Workspace needed by rl_logprob_fwd / rl_policy_loss_fwd_bwd / the split
 * phases for this shape. dz_chunk_rows = rows of the bf16 dU buffer (0 = T).
 * Includes the probability cache of rl_policy_loss_fwd_bwd[_hostio] (K1 stores
 * fp16 softmax numerators and per-32-column maxima, T x V_local x 2.125 bytes,
 * so that K4 needs no second LM-head GEMM) unless the environment sets
 * RL_P_CACHE=0 or the cache would exceed 64 GB. */
size_t rl_workspace_bytes(const rl_lm_shape* shape, int32_t num_rollouts, int64_t dz_chunk_rows);
size_t rl_workspace_bytes_hostio(const rl_lm_shape* shape, int32_t num_rollouts, int64_t dz_chunk_rows);

/* Default dU chunk rows used when dz_chunk_rows == 0 (currently T). */
int64_t rl_default_dz_chunk_rows(const rl_lm_shape* shape);

const char* rl_status_string(rl_status s);
const char* rl_last_error_message(void); /* thread-local, last failing call */
int32_t rl_abi_version(void);

/* Number of kernels the last successful call on this thread enqueued
 * (reported as gpu_launches by bench.py). */
int32_t rl_last_launch_count(void);

/* ------------------------------------------------- kernel timing (bench) */
/* When enabled (per host thread), every kernel that later calls enqueue is
 * bracketed by two CUDA events recorded on the call's stream. rl_profile_read
 * waits for the recorded events, writes up to `cap` entries (kernel id +
 * milliseconds, in launch order), clears the record and returns how many
 * launches were recorded (which may exceed cap). Timing adds two event records
 * per launch and nothing else; it is off by default. */
typedef enum rl_kernel_id {
  RL_K_GROUP_ADV = 0,  /* K0 S0                                  */
  RL_K_FWD_GEMM = 1,   /* K1 S1+S2 tile partials (tcgen05)       */
  RL_K_MERGE = 2,      /* K2 S2 merge                            */
  RL_K_LOSS = 3,       /* K3 S3 per-rollout coef + counters      */
  RL_K_FINALIZE = 4,   /* K3b report reduction                   */
  RL_K_DZ_GEMM = 5,    /* K4 S4 recompute + dU (tcgen05)         */
  RL_K_DH_GEMM = 6,    /* K5 S5 dH = dU W (tcgen05)              */
  RL_K_DW_GEMM = 7,    /* K6 S6 dW (+)= dU^T h (tcgen05)         */
  RL_K_MEMSET = 8,     /* zero fill of an empty batch's dW       */
  RL_K_NS_GEMM = 9,    /* Newton-Schulz / Muon GEMMs (tcgen05)   */
  RL_K_NS_AUX = 10,    /* Newton-Schulz / Muon SIMT kernels      */
  RL_K_GROUPED_GEMM = 11, /* MoE grouped GEMM (tcgen05)          */
  RL_K_COMPACT = 12,   /* sparse-backward compaction / gather / scatter */
  RL_K_DZ_CACHE = 13   /* K4 S4 dU from K1's probability cache (elementwise, HBM-bound) */
} rl_kernel_id;

typedef struct rl_kernel_time {
  int32_t kernel; /* rl_kernel_id */
  float ms;
} rl_kernel_time;

rl_status rl_profile_enable(int32_t enable);
int32_t rl_profile_read(rl_kernel_time* out, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* RL_H_ */
