"""Seeded synthetic rollout batches shaped like the paper's RL workload.

This module is the ONE piece shared by the oracle side (tests, `bench.py
--impl reference`) and the CUDA side (tests, `bench.py`). It holds none of the
method's arithmetic: no logits, no softmax, no ratio, no mask, no advantage.
It only draws random inputs with the shapes and distributions DESIGN.md §3
states. The one derived input, `infer_logprobs`, needs a reference log-prob
from whichever side is under test; `compose_infer_logprobs` only subtracts the
drawn noise from it and clamps at 0 (SPEC TokenRecord: infer_logprob <= 0).

Workload shapes follow BASELINE.json `configs`; the paper's RL run uses groups
of G=16 rollouts per prompt (§3.3) and binary rewards
(§3.1, "rewards it with 1 for a correct answer and 0").

Streams: one numpy PCG64 stream per tensor, keyed `[seed, k]`, so every
tensor is reproducible on any platform and independent of the others.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# stream keys, one per drawn tensor
_K_HIDDEN, _K_W, _K_TARGETS, _K_REWARDS, _K_DELTA, _K_LENGTHS, _K_SPIKES, _K_MASK, _K_SAMPLE = range(9)

# 2: adds `sample_u` (uniforms for sampling targets from the policy)
GENERATOR_VERSION = 2


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json config. Sizes are per rank unless `n_ranks` > 1."""

    name: str
    num_prompts: int          # Np
    group_size: int           # G (rollouts per prompt)
    rollout_len: int          # mean packed length of one rollout (prompt + completion)
    hidden: int               # H
    vocab: int                # V (global)
    sigma_z: float = 4.0      # std of a logit z = h.w (controls entropy)
    delta_sigma: float = 0.3  # std of the trainer-inference log-prob mismatch
    spike_rate: float = 1e-5  # per-token probability of a guard spike (infer := 0)
    prompt_frac: float = 0.0  # leading fraction of every rollout with loss_mask = 0
    ragged: bool = False      # lognormal rollout lengths instead of equal ones
    inv_temperature: float = 1.0
    n_ranks: int = 1          # ranks the config is meant for (informational)

    @property
    def num_rollouts(self) -> int:
        return self.num_prompts * self.group_size

    @property
    def tokens(self) -> int:
        return self.num_rollouts * self.rollout_len


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": Workload("tiny", 2, 4, 64, 64, 1024),
    "small": Workload("small", 8, 8, 2048, 2048, 32000),
    "glm16k": Workload("glm16k", 1, 16, 1024, 4096, 151552),
    "glm64k": Workload("glm64k", 1, 16, 4096, 4096, 151552, n_ranks=8),
    "stress": Workload("stress", 8, 16, 1024, 4096, 151552, delta_sigma=1.0,
                       spike_rate=1e-4, n_ranks=8),
}

# paper constants
ALPHA = 0.5
BETA = 5.0
GUARD = 1e-5


def _rng(seed: int, key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), int(key)]))


def float32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even); returns uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def _normal_bf16(rng: np.random.Generator, rows: int, cols: int, std: float,
                 chunk_rows: int = 8192) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.uint16)
    for r0 in range(0, rows, chunk_rows):
        r1 = min(rows, r0 + chunk_rows)
        x = rng.standard_normal((r1 - r0, cols), dtype=np.float32)
        if std != 1.0:
            x *= np.float32(std)
        out[r0:r1] = float32_to_bf16_bits(x)
    return out


def rollout_lengths(wl: Workload, seed: int, total_tokens: int | None = None) -> np.ndarray:
    """Per-rollout packed lengths summing to T (equal, or lognormal sigma=1 when ragged)."""
    R = wl.num_rollouts
    T = wl.tokens if total_tokens is None else total_tokens
    if not wl.ragged:
        base = np.full(R, T // R, dtype=np.int64)
        base[: T - int(base.sum())] += 1
        return base
    w = _rng(seed, _K_LENGTHS).lognormal(0.0, 1.0, size=R)
    lo = 1 if T >= R else 0          # fewer tokens than rollouts: some rollouts are empty
    L = np.maximum(lo, np.floor(w / w.sum() * T).astype(np.int64))
    # fix the rounding so the lengths sum to exactly T (largest rollouts absorb it)
    diff = T - int(L.sum())
    order = np.argsort(-L, kind="stable")
    i = 0
    while diff != 0:
        j = order[i % R]
        step = 1 if diff > 0 else -1
        if L[j] + step >= lo:
            L[j] += step
            diff -= step
        i += 1
    return L


def group_rewards(wl: Workload, seed: int) -> np.ndarray:
    """Binary rewards [Np, G]; a group is redrawn until it is non-constant, as the
    paper's online filter drops groups that are always solved or always failed
    (§2.1.5)."""
    rng = _rng(seed, _K_REWARDS)
    S = np.empty((wl.num_prompts, wl.group_size), dtype=np.float32)
    for p in range(wl.num_prompts):
        while True:
            s = (rng.random(wl.group_size) < 0.5).astype(np.float32)
            if s.min() != s.max():
                break
        S[p] = s
    return S


@dataclasses.dataclass
class Batch:
    wl: Workload
    seed: int
    hidden: np.ndarray           # [T, H] uint16 (bf16 bits), row-major
    w_vocab: np.ndarray          # [V, H] uint16 (bf16 bits), nn.Linear layout
    targets: np.ndarray          # [T] int32 in [0, V)
    rewards: np.ndarray          # [Np, G] float32
    rollout_offsets: np.ndarray  # [R+1] int32, CSR over the packed rows
    loss_mask: np.ndarray        # [T] uint8
    delta_noise: np.ndarray      # [T] float64, trainer-minus-inference log-prob noise
    spikes: np.ndarray           # [T] bool, positions whose stored infer log-prob is 0
    sample_u: np.ndarray         # [T] float64 uniforms in [0, 1): the draw that picks y_t when the
                                 # targets are sampled from the policy (tests/harness.py); `targets`
                                 # above is the uniform-id fallback

    @property
    def T(self) -> int:
        return int(self.hidden.shape[0])

    @property
    def H(self) -> int:
        return int(self.hidden.shape[1])

    @property
    def V(self) -> int:
        return int(self.w_vocab.shape[0])

    @property
    def loss_denominator(self) -> float:
        """D = sum_i |y_i| of Eq.1: the number of loss tokens (reading R5)."""
        return float(int(self.loss_mask.sum()))


def make_batch(wl: Workload, seed: int = 0, *, tokens: int | None = None,
               vocab: int | None = None, hidden: int | None = None,
               with_weights: bool = True, w_seed: int | None = None) -> Batch:
    """Draw one packed micro-batch. `tokens`, `vocab`, `hidden` override the config
    sizes (used for the ragged parity cases and the bounded CPU samples)."""
    T = wl.tokens if tokens is None else int(tokens)
    V = wl.vocab if vocab is None else int(vocab)
    H = wl.hidden if hidden is None else int(hidden)
    if H <= 0 or V <= 0 or T < 0:
        raise ValueError("bad sizes")
    hid = _normal_bf16(_rng(seed, _K_HIDDEN), T, H, 1.0)
    ws = seed if w_seed is None else w_seed
    W = (_normal_bf16(_rng(ws, _K_W), V, H, wl.sigma_z / math.sqrt(H)) if with_weights
         else np.zeros((0, H), dtype=np.uint16))
    targets = _rng(seed, _K_TARGETS).integers(0, V, size=T, dtype=np.int64).astype(np.int32)
    S = group_rewards(wl, seed)
    L = rollout_lengths(wl, seed, T)
    offsets = np.zeros(wl.num_rollouts + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(L)
    lm = np.ones(T, dtype=np.uint8)
    if wl.prompt_frac > 0:
        for i in range(wl.num_rollouts):
            a, b = int(offsets[i]), int(offsets[i + 1])
            lm[a: a + int(math.floor(wl.prompt_frac * (b - a)))] = 0
    delta = _rng(seed, _K_DELTA).normal(0.0, wl.delta_sigma, size=T)
    spikes = _rng(seed, _K_SPIKES).random(T) < wl.spike_rate
    u = _rng(seed, _K_SAMPLE).random(T)
    return Batch(wl, seed, hid, W, targets, S, offsets.astype(np.int32), lm, delta, spikes, u)


def compose_infer_logprobs(logp_ref: np.ndarray, delta_noise: np.ndarray,
                           spikes: np.ndarray) -> np.ndarray:
    """Stored inference log-probs: infer = min(0, logp_ref - delta); spikes get 0.

    `logp_ref` comes from the side under test's own reference (the oracle in the
    parity tests). A spike sets the stored log-prob to 0 (probability 1), so the
    token's ratio is exp(logp_ref), far below the 1e-5 guard for any target whose
    trainer log-prob is below ln 1e-5."""
    x = np.minimum(0.0, np.asarray(logp_ref, dtype=np.float64) - delta_noise)
    x = np.where(spikes, 0.0, x)
    return x.astype(np.float32)


def bf16_bits_to_float32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32 (for building device tensors)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ----------------------------------------------------------- device-side draw
def make_batch_device(wl: Workload, seed: int = 0, *, device="cuda", tokens: int | None = None,
                      vocab: int | None = None, vocab_offset: int = 0, vocab_total: int | None = None,
                      w_seed: int = 12345):
    """The same recipe as make_batch, drawn with torch's device generator (fast at
    GLM sizes; used by bench.py, whose timed numbers need no oracle parity).
    W rows [vocab_offset, vocab_offset + vocab) of a (vocab_total x H) matrix drawn
    from `w_seed` (identical on every rank). Returns a dict of device tensors plus
    host-side rewards/offsets/loss mask and the Delta noise / spikes as tensors."""
    import torch

    T = wl.tokens if tokens is None else int(tokens)
    Vt = wl.vocab if vocab_total is None else int(vocab_total)
    V = Vt - vocab_offset if vocab is None else int(vocab)
    H = wl.hidden
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 7919 + 1)
    hidden = torch.empty(T, H, dtype=torch.bfloat16, device=device)
    for r0 in range(0, T, 8192):
        r1 = min(T, r0 + 8192)
        hidden[r0:r1] = torch.randn(r1 - r0, H, generator=g, device=device).to(torch.bfloat16)
    gw = torch.Generator(device=device)
    std = wl.sigma_z / math.sqrt(H)
    w = torch.empty(V, H, dtype=torch.bfloat16, device=device)
    # draw the full matrix block by block so every shard sees the same rows
    blk = 8192
    for b0 in range(0, Vt, blk):
        b1 = min(Vt, b0 + blk)
        lo, hi = max(b0, vocab_offset), min(b1, vocab_offset + V)
        if lo >= hi:
            continue
        gw.manual_seed(int(w_seed) * 1000003 + b0)
        x = torch.randn(b1 - b0, H, generator=gw, device=device) * std
        w[lo - vocab_offset: hi - vocab_offset] = x[lo - b0: hi - b0].to(torch.bfloat16)
    targets = torch.randint(0, Vt, (T,), generator=g, device=device, dtype=torch.int64).to(torch.int32)
    S = group_rewards(wl, seed)
    L = rollout_lengths(wl, seed, T)
    offsets = np.zeros(wl.num_rollouts + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(L)
    lm = np.ones(T, dtype=np.uint8)
    if wl.prompt_frac > 0:
        for i in range(wl.num_rollouts):
            a, b = int(offsets[i]), int(offsets[i + 1])
            lm[a: a + int(math.floor(wl.prompt_frac * (b - a)))] = 0
    delta = torch.randn(T, generator=g, device=device, dtype=torch.float32) * wl.delta_sigma
    spikes = torch.rand(T, generator=g, device=device) < wl.spike_rate
    return dict(hidden=hidden, w=w, targets=targets, rewards=S.reshape(-1).copy(),
                offsets=offsets.astype(np.int32), loss_mask=lm, delta=delta, spikes=spikes)
