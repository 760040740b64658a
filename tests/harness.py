"""Shared test plumbing: build one synthetic batch, run the fp64 oracle on it, run
the CUDA path through the C ABI on the same bytes, and compare at the north-star
tolerances (BASELINE.json): log-probs and loss within 2e-3 absolute, gradients
within 1e-2 relative Frobenius error, the token mask bit-exact except for tokens
whose oracle ratio lies within 1e-4 of a masking bound (reading R13)."""
from __future__ import annotations

import dataclasses

import numpy as np

import oracle
import synth

LOGP_TOL = 2e-3
LOSS_TOL = 2e-3
GRAD_RTOL = 1e-2
BAND = 1e-4


@dataclasses.dataclass
class Case:
    batch: synth.Batch
    h64: np.ndarray
    w64: np.ndarray
    infer: np.ndarray        # float32 stored inference log-probs
    adv: np.ndarray          # [R] float32 advantages (oracle fp64 rounded; S0 is tested separately)
    inv_temperature: object    # scalar 1/tau, or a [T] float64 array (per-token, R20)
    alpha: float = synth.ALPHA
    beta: float = synth.BETA
    guard: float = synth.GUARD
    variant: str = "icepop"
    kl_tau: float = 0.0          # R19
    kl_set: str = "masked"


def make_case(wl: synth.Workload, seed=0, *, tokens=None, vocab=None, hidden=None, inv_temperature=1.0,
              corrupt=None) -> Case:
    b = synth.make_batch(wl, seed, tokens=tokens, vocab=vocab, hidden=hidden)
    h64, w64 = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h64, w64, inv_temperature)
    logp_ref, _, _ = oracle.log_softmax_stats(Z, b.targets)
    infer = synth.compose_infer_logprobs(logp_ref, b.delta_noise, b.spikes)
    if corrupt is not None:
        corrupt(b, infer)
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    return Case(b, h64, w64, infer, adv, inv_temperature)


def run_oracle(c: Case, backward=True, loss_denominator=None):
    b = c.batch
    return oracle.policy_loss_fwd_bwd(
        c.h64, c.w64, b.targets, c.infer.astype(np.float64), None, b.rollout_offsets, b.loss_mask,
        alpha=c.alpha, beta=c.beta, guard_threshold=c.guard,
        loss_denominator=b.loss_denominator if loss_denominator is None else loss_denominator,
        inv_temperature=c.inv_temperature, backward=backward, rollout_adv=c.adv.astype(np.float64),
        variant=c.variant, kl_tau=c.kl_tau, kl_set=c.kl_set)


def band_tokens(c: Case, ref) -> np.ndarray:
    if c.variant == "gspo":
        # the gate is per rollout: s_i = exp(mean log k) within 1e-4 of a clip bound
        b = c.batch
        v = ref.report.valid
        R = len(b.rollout_offsets) - 1
        rollout_of = np.repeat(np.arange(R), np.diff(b.rollout_offsets))
        lr = np.where(v, ref.logp - c.infer.astype(np.float64), 0.0)
        n = np.bincount(rollout_of, weights=v.astype(float), minlength=R)
        s = np.exp(np.bincount(rollout_of, weights=lr, minlength=R) / np.maximum(n, 1))
        near = (np.abs(s - c.alpha) <= BAND) | (np.abs(s - c.beta) <= BAND)
        return v & near[rollout_of]
    k = ref.report.ratio
    v = ref.report.valid
    near = (np.abs(k - c.alpha) <= BAND) | (np.abs(k - c.beta) <= BAND)
    if c.guard > 0:
        near |= np.abs(k / c.guard - 1.0) <= BAND
    return v & near


def rel_fro(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def compare(c: Case, ref, gpu: dict, check_grads=True) -> dict:
    """gpu: dict of numpy arrays: logprob, entropy, lse, coef, keep, guarded, report (dict),
    d_hidden, d_w_vocab. Asserts the contract; returns the measured errors."""
    b = c.batch
    err = {}
    err["logprob"] = float(np.max(np.abs(gpu["logprob"] - ref.logp))) if b.T else 0.0
    assert err["logprob"] <= LOGP_TOL, err
    if "entropy" in gpu:
        err["entropy"] = float(np.max(np.abs(gpu["entropy"] - ref.entropy))) if b.T else 0.0
        assert err["entropy"] <= LOGP_TOL, err
    if "lse" in gpu:
        err["lse"] = float(np.max(np.abs(gpu["lse"] - ref.lse))) if b.T else 0.0
        assert err["lse"] <= LOGP_TOL, err
    rep = gpu["report"]
    err["loss"] = abs(rep["loss"] - ref.report.loss)
    assert err["loss"] <= LOSS_TOL, (rep["loss"], ref.report.loss)
    band = band_tokens(c, ref)
    flips = np.nonzero(gpu["keep"].astype(bool) != ref.report.keep)[0]
    err["keep_flips"] = int(len(flips))
    assert np.all(band[flips]), f"keep flips outside the 1e-4 band at {flips[~band[flips]][:10]}"
    rollout_of = np.repeat(np.arange(len(c.adv)), np.diff(b.rollout_offsets))
    band_rollouts = np.zeros(len(c.adv), bool)
    np.logical_or.at(band_rollouts, rollout_of[band], True) if band.any() else None
    gflips = np.nonzero(gpu["guarded"].astype(bool) != ref.report.guarded)[0]
    assert np.all(band_rollouts[gflips]), f"guard flips outside the band: {gflips}"
    nband = int(band.sum())
    for key in ("kept_tokens", "masked_low", "masked_high", "guarded_tokens", "guarded_rollouts"):
        ref_v = getattr(ref.report, key)
        slack = nband if key != "guarded_tokens" else int(np.diff(b.rollout_offsets)[band_rollouts].sum())
        if key == "guarded_rollouts":
            slack = int(band_rollouts.sum())
        assert abs(rep[key] - ref_v) <= slack, (key, rep[key], ref_v)
    for key in ("nonfinite_inputs", "bad_targets", "bad_offsets"):
        assert rep[key] == getattr(ref.report, key), (key, rep[key], getattr(ref.report, key))
    if ref.report.valid.any():
        err["kl"] = abs(rep["mismatch_kl_sum"] - ref.report.mismatch_kl_sum) / max(1.0, abs(ref.report.mismatch_kl_sum))
        assert err["kl"] <= 1e-3, err
    if "coef" in gpu:
        both = gpu["keep"].astype(bool) & ref.report.keep
        if both.any():
            ce = np.abs(gpu["coef"][both] - ref.report.coef[both]) / np.maximum(np.abs(ref.report.coef[both]), 1e-30)
            err["coef_rel"] = float(ce.max())
            assert err["coef_rel"] <= 1e-2, err
    if check_grads:
        if gpu.get("d_hidden") is not None:
            err["d_hidden"] = rel_fro(gpu["d_hidden"], ref.d_hidden)
            assert err["d_hidden"] <= GRAD_RTOL, err
        if gpu.get("d_w_vocab") is not None:
            err["d_w_vocab"] = rel_fro(gpu["d_w_vocab"], ref.d_w_vocab)
            assert err["d_w_vocab"] <= GRAD_RTOL, err
    return err


# ------------------------------------------------------------- GPU side
def to_device(c: Case, device="cuda"):
    import torch
    b = c.batch

    def bf(x):
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(device)

    return dict(
        hidden=bf(b.hidden), w=bf(b.w_vocab),
        targets=torch.from_numpy(b.targets).to(device),
        infer=torch.from_numpy(c.infer).to(device),
        adv=torch.from_numpy(c.adv).to(device),
        offsets=torch.from_numpy(b.rollout_offsets).to(device),
        loss_mask=torch.from_numpy(b.loss_mask).to(device),
        rewards=torch.from_numpy(b.rewards.reshape(-1).copy()).to(device),
    )


def run_gpu_step(c: Case, *, dh_f32=False, accumulate_dw=False, dw_init=None, use_mask=True, device="cuda",
                 loss_denominator=None, dense_backward=False, dz_chunk_rows=0):
    import torch
    import paper_2512_16144_b200 as rl
    b = c.batch
    d = to_device(c, device)
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    if np.ndim(c.inv_temperature) == 1:
        invt = torch.from_numpy(np.asarray(c.inv_temperature, dtype=np.float32)).to(device)
        shape = rl.make_shape(T, H, V, 0, V, 1.0, inv_temperature_rows=invt)
    else:
        shape = rl.make_shape(T, H, V, 0, V, c.inv_temperature)
    params = rl.make_params(R, b.loss_denominator if loss_denominator is None else loss_denominator,
                            c.alpha, c.beta, c.guard, c.variant, kl_tau=c.kl_tau, kl_set=c.kl_set)
    f32 = dict(dtype=torch.float32, device=device)
    out = dict(logprob=torch.empty(T, **f32), entropy=torch.empty(T, **f32), lse=torch.empty(T, **f32),
               coef=torch.empty(T, **f32), keep=torch.empty(T, dtype=torch.uint8, device=device),
               guarded=torch.empty(R, dtype=torch.uint8, device=device))
    report = rl.new_report(device)
    dh = torch.empty(T, H, **f32) if dh_f32 else torch.empty(T, H, dtype=torch.bfloat16, device=device)
    dw = (dw_init.clone() if dw_init is not None else torch.empty(V, H, **f32))
    rl.rl_policy_loss_fwd_bwd(shape, params, d["hidden"], d["w"], d["targets"], d["infer"], d["adv"], d["offsets"],
                              d["loss_mask"] if use_mask else None, report=report, logprob=out["logprob"],
                              entropy=out["entropy"], lse=out["lse"], coef=out["coef"], token_keep=out["keep"],
                              rollout_guarded=out["guarded"], d_hidden=None if dh_f32 else dh,
                              d_hidden_f32=dh if dh_f32 else None, d_w_vocab=dw, accumulate_dw=accumulate_dw,
                              dense_backward=dense_backward, dz_chunk_rows=dz_chunk_rows)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["report"] = rl.read_report(report).as_dict()
    res["d_hidden"] = dh.float().cpu().numpy().astype(np.float64)
    res["d_w_vocab"] = dw.cpu().numpy().astype(np.float64)
    res["launches"] = rl.rl_last_launch_count()
    return res
