"""Plain fp64 CPU oracle for the IcePop policy-loss step (TEST INFRASTRUCTURE).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module. The product path
(`paper_2512_16144_b200`, `librl`) never does, and this module imports
nothing from it.

Each function restates one step of PAPER.md §3.3 (lines 449-472) in fp64:

  Eq.1 (L451-463)  J = E[ 1/sum_i|y_i| * sum_i sum_t M(pi_train/pi_infer; a, b) * A_it ]
  Eq.2 (L465-468)  M(k) = k if k in [a, b] else 0
  L470             A_it = S_i - mean({S_j} over the G rollouts of the prompt), a=0.5, b=5
  L472             a rollout is masked if any of its token ratios falls under 1e-5

with the readings of DESIGN.md §2 (R1-R15) wherever the paper is silent.
The method reaches an exact result with a plain definition (a log-softmax of a
matrix product, an elementwise gate, a sum), so the oracle is that definition
written out; the only library primitives are numpy's matrix product, exp, log,
max and sum.

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): SPEC example tables, closed
forms (uniform logits, two-level logits), normalisation, scipy/torch float64
library cross-checks, on-policy closed form, finite differences, autograd,
the dZ/dW row-sum invariants, bf16 decode of hand-worked bit patterns, and the
hand-summed mismatch_kl_sum of tests/golden/hand_loss_example.json.
"""
from __future__ import annotations

import dataclasses

import numpy as np


# ---------------------------------------------------------------- input decode
def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> exact float64 values."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


# ------------------------------------------------------------------ advantages
def group_advantages(S: np.ndarray) -> np.ndarray:
    """A_i = S_i - mean_G(S) per prompt group, no std division (PAPER.md L470,
    "Dr. GRPO"; reading R7). S is [Np, G]; returns [Np, G] fp64. G < 2 is
    rejected (SPEC compute_advantages: "group size < 2 rejected")."""
    S = np.asarray(S, dtype=np.float64)
    if S.ndim != 2 or S.shape[1] < 2:
        raise ValueError("group_advantages needs [num_groups, G] with G >= 2")
    return S - S.mean(axis=1, keepdims=True)


# ------------------------------------------------------------ LM head + softmax
def lm_logits(hidden: np.ndarray, w_vocab: np.ndarray, inv_temperature=1.0,
              vocab_block: int = 16384) -> np.ndarray:
    """z[t, v] = invT_t * sum_h hidden[t, h] * W[v, h]  (pi_train's logits in Eq.1;
    reading R8 for the temperature, R20 for a per-token invT_t: a scalar or a [T]
    array). Inputs are fp64 (exact bf16 values). Columns are computed a vocab
    block at a time only to bound memory; every entry is the same single dot
    product either way."""
    T, V = hidden.shape[0], w_vocab.shape[0]
    Z = np.empty((T, V), dtype=np.float64)
    for v0 in range(0, V, vocab_block):
        v1 = min(V, v0 + vocab_block)
        Z[:, v0:v1] = hidden @ w_vocab[v0:v1].T
    if np.ndim(inv_temperature) == 1:
        Z *= np.asarray(inv_temperature, dtype=np.float64)[:, None]
    elif inv_temperature != 1.0:
        Z *= inv_temperature
    return Z


def log_softmax_stats(Z: np.ndarray, targets: np.ndarray):
    """Per row t: lse_t = log sum_v exp(z_tv) (max-shifted), logp_t = z_{t,y_t} - lse_t
    (log pi_train(y_t | ...) of Eq.1), entropy_t = -sum_v p_tv log p_tv with
    p = exp(z - lse) (reading R9). Returns (logp, entropy, lse), each [T] fp64."""
    m = Z.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(Z - m).sum(axis=1, keepdims=True)))[:, 0]
    rows = np.arange(Z.shape[0])
    logp = Z[rows, targets] - lse
    P = np.exp(Z - lse[:, None])
    entropy = lse - (P * Z).sum(axis=1)
    return logp, entropy, lse


# ------------------------------------------------------------------- the gate
def masking_function(k: np.ndarray, alpha: float, beta: float) -> np.ndarray:
    """Eq.2: M(k) = k if alpha <= k <= beta else 0 (closed
    interval, reading R4/SPEC mask_ratio)."""
    k = np.asarray(k, dtype=np.float64)
    return np.where((k >= alpha) & (k <= beta), k, 0.0)


def rollout_guard(k: np.ndarray, offsets: np.ndarray, loss_mask: np.ndarray,
                  threshold: float) -> np.ndarray:
    """mask rollout i iff some loss token t of i has k_t < threshold
    (strict, reading R4). The min over a rollout with no loss token is +inf, i.e.
    not guarded. Returns bool [R]."""
    R = len(offsets) - 1
    g = np.zeros(R, dtype=bool)
    for i in range(R):
        a, b = int(offsets[i]), int(offsets[i + 1])
        sel = k[a:b][loss_mask[a:b].astype(bool)]
        g[i] = sel.size > 0 and sel.min() < threshold
    return g


def validate_offsets(offsets: np.ndarray, T: int) -> bool:
    o = np.asarray(offsets, dtype=np.int64)
    return o.ndim == 1 and o.size >= 1 and o[0] == 0 and o[-1] == T and bool(np.all(np.diff(o) >= 0))


@dataclasses.dataclass
class LossReport:
    """SPEC LossReport extended with the counters of DESIGN.md §4."""
    loss: float                 # -J (reading R3): local contribution already / D
    coef: np.ndarray            # [T] keep_t * k_t * A_i / D  (d loss / d logp_t = -coef_t)
    keep: np.ndarray            # [T] bool
    guarded: np.ndarray         # [R] bool
    ratio: np.ndarray           # [T] k_t
    valid: np.ndarray           # [T] bool (loss token with finite infer <= 0 and valid target)
    masked_low: int
    masked_high: int
    guarded_rollouts: int
    guarded_tokens: int
    kept_tokens: int
    nonfinite_inputs: int
    bad_targets: int
    bad_offsets: int
    mismatch_kl_sum: float      # sum over valid tokens of k - log k - 1


def icepop_loss(logp: np.ndarray, infer_logprobs: np.ndarray, rollout_adv: np.ndarray,
                offsets: np.ndarray, loss_mask: np.ndarray | None, alpha: float,
                beta: float, guard_threshold: float, loss_denominator: float,
                targets: np.ndarray | None = None, vocab: int | None = None) -> LossReport:
    """Eq.1 + Eq.2 + the rollout guard, step by step (DESIGN.md §2 R1-R6, R10):

      k_t     = exp(logp_t - infer_t)                           (Eq.1 ratio)
      valid_t = loss_mask_t and infer_t finite and <= 0 and y_t in [0, V)
      g_i     = min_{t in i, valid} k_t < guard                  (L472)
      keep_t  = valid_t and alpha <= k_t <= beta and not g_i     (Eq.2)
      coef_t  = keep_t ? k_t * A_i / D : 0
      loss    = -sum_t coef_t                                    (minimise -J)
    """
    T = len(logp)
    logp = np.asarray(logp, dtype=np.float64)
    infer = np.asarray(infer_logprobs, dtype=np.float64)
    A = np.asarray(rollout_adv, dtype=np.float64)
    lm = np.ones(T, dtype=bool) if loss_mask is None else np.asarray(loss_mask).astype(bool)
    if loss_denominator <= 0:
        raise ValueError("loss_denominator must be > 0")
    R = len(offsets) - 1
    if not validate_offsets(offsets, T) or len(A) != R:
        # malformed packing: the whole batch is neutralised
        z = np.zeros(T)
        return LossReport(0.0, z, np.zeros(T, bool), np.zeros(max(R, 0), bool), z.copy(),
                          np.zeros(T, bool), 0, 0, 0, 0, 0, 0, 0, 1, 0.0)
    finite_ok = np.isfinite(infer) & (infer <= 0.0)
    tgt_ok = np.ones(T, dtype=bool)
    if targets is not None and vocab is not None:
        tgt_ok = (targets >= 0) & (targets < vocab)
    valid = lm & finite_ok & tgt_ok
    with np.errstate(invalid="ignore", over="ignore"):
        delta = np.where(valid, logp - infer, 0.0)
    k = np.exp(delta)
    g = rollout_guard(k, offsets, valid, guard_threshold)
    rollout_of = np.repeat(np.arange(R), np.diff(np.asarray(offsets, dtype=np.int64)))
    M = masking_function(k, alpha, beta)
    in_band = M > 0
    keep = valid & in_band & ~g[rollout_of]
    coef = np.where(keep, k * A[rollout_of] / loss_denominator, 0.0)
    loss = -coef.sum()
    return LossReport(
        loss=float(loss), coef=coef, keep=keep, guarded=g, ratio=k, valid=valid,
        masked_low=int((valid & (k < alpha)).sum()),
        masked_high=int((valid & (k > beta)).sum()),
        guarded_rollouts=int(g.sum()),
        guarded_tokens=int((valid & g[rollout_of]).sum()),
        kept_tokens=int(keep.sum()),
        nonfinite_inputs=int((lm & ~finite_ok).sum()),
        bad_targets=int((lm & finite_ok & ~tgt_ok).sum()),
        bad_offsets=0,
        mismatch_kl_sum=float(np.where(valid, k - delta - 1.0, 0.0).sum()),
    )


# ------------------------------------------------------- loss variants (§8 f2)
def _segments(offsets, T):
    R = len(offsets) - 1
    return R, np.repeat(np.arange(R), np.diff(np.asarray(offsets, dtype=np.int64)))


def cispo_loss(logp, infer_logprobs, rollout_adv, offsets, loss_mask, clip_low, clip_high, guard_threshold,
               loss_denominator, targets=None, vocab=None) -> LossReport:
    """CISPO (MiniMax-M1, cited at PAPER.md L472: "similar to CISPO ... we use masking
    instead of clipping"; reading R16): the ratio is clipped, not masked, and enters as a
    stop-gradient weight on log pi_train:

      J      = 1/D sum_t valid_t (1 - g_i) sg(clip(k_t, lo, hi)) A_i logp_t
      coef_t = valid_t (1 - g_i) clip(k_t, lo, hi) A_i / D          (d(-J)/d logp_t = -coef_t)
      loss   = -sum_t coef_t logp_t
    The rollout guard of L472 still applies (guard_threshold = 0 disables it).
    masked_low / masked_high count tokens whose ratio was clipped."""
    T = len(logp)
    base = icepop_loss(logp, infer_logprobs, rollout_adv, offsets, loss_mask, 0.0, np.inf, guard_threshold,
                       loss_denominator, targets, vocab)
    if base.bad_offsets:
        return base
    R, rollout_of = _segments(offsets, T)
    k = base.ratio
    valid = base.valid
    keep = valid & ~base.guarded[rollout_of]
    w = np.clip(k, clip_low, clip_high)
    coef = np.where(keep, w * np.asarray(rollout_adv, np.float64)[rollout_of] / loss_denominator, 0.0)
    loss = -float((coef * np.where(keep, logp, 0.0)).sum())
    return dataclasses.replace(base, loss=loss, coef=coef, keep=keep,
                               masked_low=int((valid & (k < clip_low)).sum()),
                               masked_high=int((valid & (k > clip_high)).sum()),
                               kept_tokens=int(keep.sum()))


def gspo_loss(logp, infer_logprobs, rollout_adv, offsets, loss_mask, clip_low, clip_high, guard_threshold,
              loss_denominator, targets=None, vocab=None) -> LossReport:
    """GSPO (Qwen, the sequence-level objective of PAPER.md Fig. 8; reading R17):

      s_i    = exp( (1/n_i) sum_{t in i, valid} (logp_t - infer_t) )      (n_i valid tokens)
      J      = 1/D sum_i [n_i > 0] (1 - g_i) min(s_i A_i, clip(s_i, lo, hi) A_i)
      coef_t = valid_t (1 - g_i) u_i s_i A_i / (n_i D),  u_i = 1 unless the min picks the
               clipped term (A_i > 0 and s_i > hi, or A_i < 0 and s_i < lo), then 0
      loss   = -J
    (d s_i / d logp_t = s_i / n_i, so d(-J)/d logp_t = -coef_t.) D is the caller's
    denominator (the GSPO paper averages over sequences: pass the rollout count).
    masked_low / masked_high count tokens of rollouts whose gradient the clip removed."""
    T = len(logp)
    base = icepop_loss(logp, infer_logprobs, rollout_adv, offsets, loss_mask, 0.0, np.inf, guard_threshold,
                       loss_denominator, targets, vocab)
    if base.bad_offsets:
        return base
    R, rollout_of = _segments(offsets, T)
    A = np.asarray(rollout_adv, np.float64)
    valid = base.valid
    with np.errstate(invalid="ignore"):
        logratio = np.where(valid, np.asarray(logp, np.float64) - np.asarray(infer_logprobs, np.float64), 0.0)
    n = np.bincount(rollout_of, weights=valid.astype(np.float64), minlength=R)
    sum_lr = np.bincount(rollout_of, weights=logratio, minlength=R)
    s = np.exp(np.divide(sum_lr, n, out=np.zeros(R), where=n > 0))
    live = (n > 0) & ~base.guarded
    clipped_hi = (A > 0) & (s > clip_high)
    clipped_lo = (A < 0) & (s < clip_low)
    u = live & ~clipped_hi & ~clipped_lo
    J = np.where(live, np.minimum(s * A, np.clip(s, clip_low, clip_high) * A), 0.0).sum() / loss_denominator
    per_rollout = np.where(u, s * A / np.where(n > 0, n, 1.0) / loss_denominator, 0.0)
    keep = valid & u[rollout_of]
    coef = np.where(keep, per_rollout[rollout_of], 0.0)
    return dataclasses.replace(base, loss=-float(J), coef=coef, keep=keep,
                               masked_low=int((valid & (live & clipped_lo)[rollout_of]).sum()),
                               masked_high=int((valid & (live & clipped_hi)[rollout_of]).sum()),
                               kept_tokens=int(keep.sum()))


LOSS_VARIANTS = {"icepop": 0, "cispo": 1, "gspo": 2}


def variant_loss(variant, *args, **kw) -> LossReport:
    """Dispatch by name: icepop (Eq.1/Eq.2, alpha/beta = mask bounds), cispo or gspo
    (alpha/beta = clip bounds)."""
    fn = {"icepop": icepop_loss, "cispo": cispo_loss, "gspo": gspo_loss}[variant]
    return fn(*args, **kw)


KL_SETS = {"masked": 0, "unmasked": 1, "all": 2}


def add_kl_term(rep: LossReport, logp, infer_logprobs, kl_tau: float, kl_set: str,
                loss_denominator: float) -> LossReport:
    """Reading R19 (not in Eq.1, default kl_tau = 0): the trainer's
    KL term on the token log-ratio,

      loss += (kl_tau / D) * sum_{t in S} log k_t,   log k_t = logp_t - infer_t,
      S = valid & ~keep ("masked"), keep ("unmasked") or valid ("all"),

    with S fixed by the gate (no gradient through it). d loss / d logp_t gains
    kl_tau / D on S, so coef_t (d loss / d logp_t = -coef_t) loses kl_tau / D."""
    if kl_tau == 0.0:
        return rep
    logp = np.asarray(logp, dtype=np.float64)
    infer = np.asarray(infer_logprobs, dtype=np.float64)
    S = {"masked": rep.valid & ~rep.keep, "unmasked": rep.keep, "all": rep.valid}[kl_set]
    logk = np.where(S, logp - np.where(S, infer, 0.0), 0.0)
    w = kl_tau / loss_denominator
    return dataclasses.replace(rep, loss=float(rep.loss + w * logk.sum()), coef=rep.coef - np.where(S, w, 0.0))


# ------------------------------------------------------------------- backward
def icepop_backward(Z: np.ndarray, lse: np.ndarray, targets: np.ndarray, coef: np.ndarray,
                    hidden: np.ndarray, w_vocab: np.ndarray, inv_temperature: float = 1.0):
    """Gradient of loss = -sum_t keep_t k_t A_i / D with the gate held fixed
    (hard mask, SPEC icepop_gradient; reading R2): d k_t = k_t d logp_t, so
    d loss / d u_tv = coef_t * invT * (p_tv - [v == y_t]) with u = hidden @ W^T.

      dZ = coef[:, None] * invT * (softmax(Z) - onehot(y))
      dH = dZ @ W            dW = dZ^T @ hidden
    Returns (dZ, dH, dW) in fp64."""
    P = np.exp(Z - lse[:, None])
    P[np.arange(Z.shape[0]), targets] -= 1.0
    dZ = (coef * np.asarray(inv_temperature, dtype=np.float64))[:, None] * P
    return dZ, dZ @ w_vocab, dZ.T @ hidden


# ------------------------------------------------------------ whole-step entry
@dataclasses.dataclass
class StepResult:
    logp: np.ndarray
    entropy: np.ndarray
    lse: np.ndarray
    report: LossReport
    d_hidden: np.ndarray | None
    d_w_vocab: np.ndarray | None
    advantages: np.ndarray


def policy_loss_fwd_bwd(hidden, w_vocab, targets, infer_logprobs, rewards, offsets,
                        loss_mask=None, *, alpha=0.5, beta=5.0, guard_threshold=1e-5,
                        loss_denominator=None, inv_temperature=1.0, backward=True,
                        rollout_adv=None, variant="icepop", kl_tau=0.0, kl_set="masked") -> StepResult:
    """The whole north-star step on one rank: S0 (advantages), S1-S2 (logits,
    log-softmax stats), S3 (Eq.1/Eq.2/guard), S4-S6 (backward). `hidden` and
    `w_vocab` are fp64 arrays (use bf16_to_f64 on bit patterns); `rewards` is
    [Np, G] unless `rollout_adv` is given directly."""
    T = hidden.shape[0]
    A = group_advantages(rewards).reshape(-1) if rollout_adv is None else np.asarray(rollout_adv, np.float64)
    lm = np.ones(T, dtype=np.uint8) if loss_mask is None else np.asarray(loss_mask)
    D = float(lm.astype(bool).sum()) if loss_denominator is None else float(loss_denominator)
    Z = lm_logits(hidden, w_vocab, inv_temperature)
    V = w_vocab.shape[0]
    safe_t = np.where((targets >= 0) & (targets < V), targets, 0)
    logp, ent, lse = log_softmax_stats(Z, safe_t)
    rep = variant_loss(variant, logp, infer_logprobs, A, offsets, lm, alpha, beta, guard_threshold,
                       D, targets=targets, vocab=V)
    rep = add_kl_term(rep, logp, infer_logprobs, kl_tau, kl_set, D)
    dH = dW = None
    if backward:
        _, dH, dW = icepop_backward(Z, lse, safe_t, rep.coef, hidden, w_vocab, inv_temperature)
    return StepResult(logp, ent, lse, rep, dH, dW, A)


# -------------------------------------------------- vocab shard statistics
def shard_stats(Z_shard: np.ndarray, targets: np.ndarray, vocab_offset: int):
    """Per-row statistics of one vocab shard (columns vocab_offset .. +V_s) of the
    scaled logits, from their definition:
      m = max_v z,  s = sum_v exp(z - m),  t = sum_v exp(z - m) (z - m),
      zt = z_{y} if y falls in the shard else -inf.
    Used to check a vocab-parallel partial and the merge identity."""
    m = Z_shard.max(axis=1)
    E = np.exp(Z_shard - m[:, None])
    s = E.sum(axis=1)
    t = (E * (Z_shard - m[:, None])).sum(axis=1)
    local = targets - vocab_offset
    inside = (local >= 0) & (local < Z_shard.shape[1])
    zt = np.full(len(targets), -np.inf)
    zt[inside] = Z_shard[np.nonzero(inside)[0], local[inside]]
    return m, s, t, zt


def merge_shard_stats(parts):
    """Combine shard statistics (m, s, t, zt) into (lse, entropy, z_target):
    with M = max m_j, S = sum s_j e^{m_j-M}, Tt = sum e^{m_j-M} (t_j + s_j (m_j-M)):
      lse = M + log S,  entropy = log S - Tt / S,  z_target = max_j zt_j."""
    ms = np.stack([p[0] for p in parts])
    M = ms.max(axis=0)
    S = sum(p[1] * np.exp(p[0] - M) for p in parts)
    Tt = sum(np.exp(p[0] - M) * (p[2] + p[1] * (p[0] - M)) for p in parts)
    zt = np.stack([p[3] for p in parts]).max(axis=0)
    return M + np.log(S), np.log(S) - Tt / S, zt
