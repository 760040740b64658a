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
    plants: dict = dataclasses.field(default_factory=dict)   # planted band-edge rows {row: (bound, dlog)}


# ------------------------------------------------------- realistic rollouts (§8(d))
def sample_from_policy(Z: np.ndarray, lse: np.ndarray, u: np.ndarray) -> np.ndarray:
    """y_t ~ softmax(Z_t): Eq.1 draws the rollouts from the policy (y_i ~ pi_infer,
    PAPER.md L455-456), so a realistic target is a sample of the row's own
    distribution. Inverse CDF with the seeded uniform u_t (synth):
    y_t = the first v with sum_{v' <= v} p_tv' > u_t. Z, lse from the oracle (fp64)."""
    C = np.cumsum(np.exp(Z - lse[:, None]), axis=1)
    y = (C <= (np.asarray(u) * C[:, -1])[:, None]).sum(axis=1)
    return np.minimum(y, Z.shape[1] - 1).astype(np.int32)


BAND_EPS = (1e-6, 2e-4, 1e-3)   # |ln k - ln b| of the planted tokens: inside, just outside, outside the band


def plant_band_tokens(b: synth.Batch, logp: np.ndarray, argmin_ids: np.ndarray, logp_argmin: np.ndarray,
                      targets: np.ndarray, infer: np.ndarray, alpha=synth.ALPHA, beta=synth.BETA, guard=synth.GUARD):
    """Tokens planted at the masking bounds (Eq.2, guard P:L472):
    infer_t = logp_t - (ln bnd + s eps), i.e. k_t = bnd e^{s eps}, for bnd in {alpha, beta,
    guard}, s = +-1, eps in BAND_EPS, in rollouts without a guard spike. alpha/beta plants
    go to loss rows of the first half of those rollouts whose logp is below ln alpha - 0.01
    (the stored log-prob stays <= 0); guard plants take the row's least likely target
    (argmin_ids, log-prob logp_argmin, ~ -36) in a rollout of their own in the second half. All arrays are [T]. Modifies
    targets / infer in place; returns {row: (bound, s * eps)}."""
    R = len(b.rollout_offsets) - 1
    rollout_of = np.repeat(np.arange(R), np.diff(b.rollout_offsets))
    ok = b.loss_mask.astype(bool) & ~b.spikes
    # rollouts without a guard spike, so a plant's own gate decides its outcome
    clean = np.setdiff1d(np.arange(R), rollout_of[b.spikes])
    half = max(1, len(clean) // 2)
    first, second = clean[:half], clean[half:]
    plants = {}
    ab = [(bnd, s * e) for bnd in (alpha, beta) for e in BAND_EPS for s in (-1, 1)]
    cand = np.nonzero(ok & np.isin(rollout_of, first) & (logp < np.log(alpha) - 0.01))[0]
    pick = cand[np.linspace(0, len(cand) - 1, num=min(len(ab), len(cand))).astype(int)] if len(cand) else []
    for r, (bnd, d) in zip(pick, ab):
        infer[r] = np.float32(logp[r] - (np.log(bnd) + d))
        plants[int(r)] = (bnd, d)
    if guard > 0:
        gs = [(guard, s * e) for e in BAND_EPS for s in (-1, 1)]
        for j, (bnd, d) in enumerate(gs):
            if j >= len(second):
                break
            cand = np.nonzero(ok & (rollout_of == second[j]))[0]
            if not len(cand):
                continue
            r = int(cand[len(cand) // 2])
            targets[r] = np.int32(argmin_ids[r])
            infer[r] = np.float32(logp_argmin[r] - (np.log(bnd) + d))
            plants[r] = (bnd, d)
    assert all(infer[r] <= 0 for r in plants)
    return plants


def make_case(wl: synth.Workload, seed=0, *, tokens=None, vocab=None, hidden=None, inv_temperature=1.0,
              corrupt=None, targets="uniform", plants=False) -> Case:
    """targets: "uniform" (ids drawn uniformly, the round-1 fallback) or "sampled" (y_t from
    the policy itself; spike rows get the row's least likely token, so the guard trips even
    when the sampled targets are probable). plants: tokens at the mask/guard bounds."""
    b = synth.make_batch(wl, seed, tokens=tokens, vocab=vocab, hidden=hidden)
    h64, w64 = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h64, w64, inv_temperature)
    if targets == "sampled" and b.T:
        _, _, lse = oracle.log_softmax_stats(Z, np.zeros(b.T, np.int64))
        b.targets = sample_from_policy(Z, lse, b.sample_u)
        if b.spikes.any():
            b.targets[b.spikes] = np.argmin(Z[b.spikes], axis=1).astype(np.int32)
    logp_ref, _, lse = oracle.log_softmax_stats(Z, b.targets)
    infer = synth.compose_infer_logprobs(logp_ref, b.delta_noise, b.spikes)
    planted = {}
    if plants and b.T:
        amin = np.argmin(Z, axis=1)
        planted = plant_band_tokens(b, logp_ref, amin, Z[np.arange(b.T), amin] - lse, b.targets, infer)
    if corrupt is not None:
        corrupt(b, infer)
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    c = Case(b, h64, w64, infer, adv, inv_temperature)
    c.plants = planted
    return c


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
        # the rollout guard applies to GSPO too (R17): its band counts as well
        gnear = np.abs(ref.report.ratio / c.guard - 1.0) <= BAND if c.guard > 0 else np.zeros(len(v), bool)
        return v & (near[rollout_of] | gnear)
    k = ref.report.ratio
    v = ref.report.valid
    near = (np.abs(k - c.alpha) <= BAND) | (np.abs(k - c.beta) <= BAND)
    if c.guard > 0:
        near |= np.abs(k / c.guard - 1.0) <= BAND
    return v & near


ROW_RTOL = 1e-2      # per dH row / per dW tile: the north star's 1e-2, applied locally
COND_FLOOR = 1e-4    # + this many units of the row's (tile's) onehot-term scale (see dh_row_error)


def dh_row_error(gpu_dh, ref_dh, coef, w64, targets, inv_temperature=1.0) -> float:
    """max_t ||dH_t - dH*_t|| / (ROW_RTOL ||dH*_t|| + COND_FLOOR |coef_t invT_t| ||W_{y_t}||); <= 1 passes.
    dH_t depends on row t only (dH_t = invT coef_t (E_p[W] - W_{y_t})), so every row is
    checked on its own, not through one global norm. The floor is the fp32 conditioning of
    p_{t,y} - 1 when p_{t,y} -> 1: logits carry ~|z| 2^-24 absolute error (TMEM fp32
    accumulation), so the GPU's p - 1 is good to ~1e-5 absolute, which is a large relative
    error once 1 - p_{t,y} < 1e-3, while the row's whole gradient is then that small."""
    gpu_dh = np.asarray(gpu_dh, np.float64)
    ref_dh = np.asarray(ref_dh, np.float64)
    if gpu_dh.size == 0:
        return 0.0
    invt = np.broadcast_to(np.asarray(inv_temperature, np.float64), (len(coef),))
    wy = np.linalg.norm(w64[np.asarray(targets) % w64.shape[0]], axis=1)
    floor = COND_FLOOR * np.abs(np.asarray(coef, np.float64) * invt) * wy
    den = ROW_RTOL * np.linalg.norm(ref_dh, axis=1) + floor
    num = np.linalg.norm(gpu_dh - ref_dh, axis=1)
    ok = den > 0
    assert not np.any(num[~ok] > 0), "non-zero dH rows where the oracle has coef = 0"
    return float((num[ok] / den[ok]).max()) if ok.any() else 0.0


def dw_tile_error(gpu_dw, ref_dw, coef, h64, targets, inv_temperature=1.0, row_ids=None, tile_rows=256,
                  tile_cols=512) -> float:
    """max over 256 x 512 tiles (the dW GEMM's output tiles) of ||dW - dW*||_tile /
    (ROW_RTOL ||dW*||_tile + COND_FLOOR ||O||_tile), O[v] = sum_{t: y_t = v} |coef_t invT_t| |h_t|
    (the scale of the onehot term, see dh_row_error). row_ids: the vocab rows given (a sample
    of whole rows, any subset), default all. <= 1 passes."""
    gpu_dw = np.asarray(gpu_dw, np.float64)
    ref_dw = np.asarray(ref_dw, np.float64)
    V_rows, H = ref_dw.shape
    row_ids = np.arange(V_rows) if row_ids is None else np.asarray(row_ids)
    invt = np.broadcast_to(np.asarray(inv_temperature, np.float64), (len(coef),))
    g = np.abs(np.asarray(coef, np.float64) * invt)
    O = np.zeros((V_rows, H))
    where = {int(v): i for i, v in enumerate(row_ids)}
    for t in np.nonzero(g)[0]:
        i = where.get(int(targets[t]))
        if i is not None:
            O[i] += g[t] * np.abs(h64[t])
    worst = 0.0
    tiles = row_ids // tile_rows
    for tb in np.unique(tiles):
        sel = tiles == tb
        for c0 in range(0, H, tile_cols):
            d = np.linalg.norm(gpu_dw[sel, c0:c0 + tile_cols] - ref_dw[sel, c0:c0 + tile_cols])
            den = ROW_RTOL * np.linalg.norm(ref_dw[sel, c0:c0 + tile_cols]) + COND_FLOOR * np.linalg.norm(
                O[sel, c0:c0 + tile_cols])
            if den > 0:
                worst = max(worst, d / den)
            else:
                assert d == 0
    return float(worst)


def guard_band_tokens(c: Case, ref) -> np.ndarray:
    """Valid tokens whose oracle ratio is within 1e-4 (relative) of the guard threshold."""
    if c.guard <= 0:
        return np.zeros(len(ref.logp), bool)
    return ref.report.valid & (np.abs(ref.report.ratio / c.guard - 1.0) <= BAND)


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
    band = band_tokens(c, ref)
    rollout_of = np.repeat(np.arange(len(c.adv)), np.diff(b.rollout_offsets))
    # a guard-band token (k within 1e-4 of tau_g, relative) may flip its rollout's guard,
    # and with it the gate of every token of that rollout (reading R13)
    gband = guard_band_tokens(c, ref)
    gband_rollouts = np.zeros(len(c.adv), bool)
    if gband.any():
        np.logical_or.at(gband_rollouts, rollout_of[gband], True)
    allowed = band | gband_rollouts[rollout_of] if b.T else band
    flips = np.nonzero(gpu["keep"].astype(bool) != ref.report.keep)[0]
    err["keep_flips"] = int(len(flips))
    assert np.all(allowed[flips]), f"keep flips outside the 1e-4 band at {flips[~allowed[flips]][:10]}"
    gflips = np.nonzero(gpu["guarded"].astype(bool) != ref.report.guarded)[0]
    err["guard_flips"] = int(len(gflips))
    assert np.all(gband_rollouts[gflips]), f"guard flips outside the band: {gflips}"
    # the loss is unique given the gate: a flipped token can move it by at most its own term
    # (|coef| for Eq.1, |coef logp| for CISPO, plus the KL term's kl_tau/D |log k|)
    slack = 0.0
    if len(flips) and "coef" in gpu:
        lk = np.abs(ref.logp[flips] - c.infer[flips].astype(np.float64))
        slack = float(((np.abs(gpu["coef"][flips]) + np.abs(ref.report.coef[flips]))
                       * np.maximum(1.0, np.abs(ref.logp[flips]))).sum()
                      + abs(c.kl_tau) / b.loss_denominator * lk.sum())
    err["loss"] = abs(rep["loss"] - ref.report.loss)
    assert err["loss"] <= LOSS_TOL + slack, (rep["loss"], ref.report.loss, slack)
    nband = int(allowed.sum())
    for key in ("kept_tokens", "masked_low", "masked_high", "guarded_tokens", "guarded_rollouts"):
        ref_v = getattr(ref.report, key)
        slack_k = nband if key != "guarded_tokens" else int(np.diff(b.rollout_offsets)[gband_rollouts].sum())
        if key == "guarded_rollouts":
            slack_k = int(gband_rollouts.sum())
        assert abs(rep[key] - ref_v) <= slack_k, (key, rep[key], ref_v)
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
    if c.plants:
        # planted band-edge tokens: outside the 1e-4 band the gate must be exact
        rows = np.array(sorted(c.plants))
        outside = rows[~band[rows]]
        err["plants_outside_band"] = int(len(outside))
        assert np.array_equal(gpu["keep"][outside].astype(bool), ref.report.keep[outside]), "planted token misclassified"
    if check_grads:
        b = c.batch
        dH_ref, dW_ref, coef_ref = ref.d_hidden, ref.d_w_vocab, ref.report.coef
        changed = np.nonzero(gpu["keep"].astype(bool) != ref.report.keep)[0]
        if len(changed) and "coef" in gpu:
            # band flips are allowed (R13); the gradient is unique GIVEN the gate, so the
            # oracle backward is re-run with the GPU's decision on the flipped rows
            coef_ref = ref.report.coef.copy()
            coef_ref[changed] = gpu["coef"][changed]
            Z = oracle.lm_logits(c.h64, c.w64, c.inv_temperature)
            safe_t = np.where((b.targets >= 0) & (b.targets < b.V), b.targets, 0)
            _, dH_ref, dW_ref = oracle.icepop_backward(Z, ref.lse, safe_t, coef_ref, c.h64, c.w64, c.inv_temperature)
        if gpu.get("d_hidden") is not None:
            err["d_hidden"] = rel_fro(gpu["d_hidden"], dH_ref)
            assert err["d_hidden"] <= GRAD_RTOL, err
            err["d_hidden_row"] = dh_row_error(gpu["d_hidden"], dH_ref, coef_ref, c.w64, b.targets, c.inv_temperature)
            assert err["d_hidden_row"] <= 1.0, err
        if gpu.get("d_w_vocab") is not None:
            err["d_w_vocab"] = rel_fro(gpu["d_w_vocab"], dW_ref)
            assert err["d_w_vocab"] <= GRAD_RTOL, err
            err["d_w_vocab_tile"] = dw_tile_error(gpu["d_w_vocab"], dW_ref, coef_ref, c.h64, b.targets,
                                                  c.inv_temperature)
            assert err["d_w_vocab_tile"] <= 1.0, err
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
                 loss_denominator=None, dense_backward=False, dz_chunk_rows=0, k0=True):
    """The whole step through the C ABI. k0: the advantages come from the rewards through
    K0 on the device (rl_group_advantages), so rewards -> K0 -> K3 is checked end to end;
    k0=False feeds the oracle's advantages (c.adv) instead."""
    import torch
    import paper_2512_16144_b200 as rl
    b = c.batch
    d = to_device(c, device)
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    if k0 and b.rewards.size == R and R > 0:
        d["adv"] = rl.rl_group_advantages(d["rewards"], b.rewards.shape[1])
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
