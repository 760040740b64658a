"""Pins of the loss-variant oracles (CISPO, GSPO; R16/R17):
hand-computed tables, relations to IcePop, closed forms, finite differences of the
actual objectives, torch autograd."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth


def _ex(golden_dir):
    base = json.load(open(os.path.join(golden_dir, "hand_loss_example.json")))
    var = json.load(open(os.path.join(golden_dir, "variant_examples.json")))
    logp = np.array(base["logp"])
    infer = logp - np.array(base["log_ratio"])
    A = oracle.group_advantages(np.array(base["rewards"], float)).reshape(-1)
    return base, var, logp, infer, A


def test_cispo_hand_example(golden_dir):
    base, var, logp, infer, A = _ex(golden_dir)
    c = var["cispo"]
    rep = oracle.cispo_loss(logp, infer, A, np.array(base["offsets"]), None, *c["clip"], 1e-5, c["D"])
    assert rep.loss == pytest.approx(c["loss"], abs=1e-12)
    np.testing.assert_allclose(rep.coef * c["D"], c["coef_times_D"], atol=1e-12)
    for k in ("masked_low", "masked_high", "kept_tokens"):
        assert getattr(rep, k) == c[k], k


def test_gspo_hand_example(golden_dir):
    base, var, logp, infer, A = _ex(golden_dir)
    g = var["gspo"]
    rep = oracle.gspo_loss(logp, infer, A, np.array(base["offsets"]), None, *g["clip"], 1e-5, g["D"])
    assert rep.loss == pytest.approx(g["loss"], abs=1e-7)
    np.testing.assert_allclose(rep.coef, g["coef"], atol=1e-7)
    for k in ("masked_low", "masked_high", "kept_tokens"):
        assert getattr(rep, k) == g[k], k


def test_cispo_equals_icepop_inside_the_band():
    """Where every ratio is inside [lo, hi], clipping and masking coincide."""
    rng = np.random.default_rng(0)
    T = 40
    logp = -rng.random(T) * 3
    infer = logp - rng.uniform(-0.3, 0.3, T)
    off = np.array([0, 10, 25, 40])
    A = np.array([0.5, -0.25, 1.0])
    a = oracle.icepop_loss(logp, infer, A, off, None, 0.5, 5.0, 1e-5, 40.0)
    b = oracle.cispo_loss(logp, infer, A, off, None, 0.5, 5.0, 1e-5, 40.0)
    np.testing.assert_allclose(a.coef, b.coef, atol=1e-15)


def test_gspo_on_policy_closed_form():
    """infer == logp: s_i = 1 and coef_t = A_i / (n_i D) for every valid token."""
    logp = np.log(np.random.default_rng(1).random(30) * 0.9 + 0.05)
    off = np.array([0, 7, 7, 30])
    A = np.array([0.3, 1.0, -0.6])
    rep = oracle.gspo_loss(logp, logp, A, off, None, 0.8, 1.25, 1e-5, 3.0)
    n = np.diff(off)
    expect = np.concatenate([np.full(n[i], A[i] / (n[i] * 3.0)) for i in range(3)])
    np.testing.assert_allclose(rep.coef, expect, atol=1e-15)
    assert rep.loss == pytest.approx(-(A[0] + A[2]) / 3.0, abs=1e-15)   # empty rollout contributes 0


def _tiny(seed, dsig=0.4):
    wl = synth.Workload("t", 2, 3, 8, 8, 16, delta_sigma=dsig, ragged=True, sigma_z=2.0, prompt_frac=0.2)
    b = synth.make_batch(wl, seed)
    h, W = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    lp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h, W), b.targets)
    infer = synth.compose_infer_logprobs(lp, b.delta_noise, b.spikes).astype(np.float64)
    return b, h, W, infer


def _gspo_objective(h, W, b, infer, A, lo, hi, D):
    """-J_GSPO(h, W) evaluated from its definition (no mask frozen: clipping is part of J)."""
    lp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h, W), b.targets)
    return oracle.gspo_loss(lp, infer, A, b.rollout_offsets, b.loss_mask, lo, hi, 0.0, D).loss


@pytest.mark.parametrize("seed,lo,hi", [(0, 0.8, 1.25), (1, 0.95, 1.05), (2, 0.5, 2.0), (3, 0.99, 1.01)])
def test_gspo_gradient_finite_differences(seed, lo, hi):
    """The sequence-level gradient coef_t = u_i s_i A_i / (n_i D) against central
    differences of the GSPO objective itself (step 1e-6, fp64)."""
    b, h, W, infer = _tiny(seed)
    A = oracle.group_advantages(b.rewards).reshape(-1)
    D = float(len(A))
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                     alpha=lo, beta=hi, guard_threshold=0.0, loss_denominator=D, variant="gspo")
    lp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h, W), b.targets)
    n = np.bincount(np.repeat(np.arange(len(A)), np.diff(b.rollout_offsets)), weights=b.loss_mask, minlength=len(A))
    sr = np.bincount(np.repeat(np.arange(len(A)), np.diff(b.rollout_offsets)),
                     weights=np.where(b.loss_mask > 0, lp - infer, 0.0), minlength=len(A))
    s = np.exp(sr / np.maximum(n, 1))
    if np.any(np.abs(s - lo) < 1e-4) or np.any(np.abs(s - hi) < 1e-4):
        pytest.skip("a sequence ratio sits on a clip bound")
    eps = 1e-6
    rng = np.random.default_rng(seed)
    for X, G in ((h, res.d_hidden), (W, res.d_w_vocab)):
        for _ in range(20):
            ix = tuple(rng.integers(0, d) for d in X.shape)
            old = X[ix]
            X[ix] = old + eps
            fp = _gspo_objective(h, W, b, infer, A, lo, hi, D)
            X[ix] = old - eps
            fm = _gspo_objective(h, W, b, infer, A, lo, hi, D)
            X[ix] = old
            assert (fp - fm) / (2 * eps) == pytest.approx(G[ix], rel=1e-5, abs=1e-10)


def test_gspo_matches_torch_autograd():
    b, h, W, infer = _tiny(4, dsig=0.05)
    A = oracle.group_advantages(b.rewards).reshape(-1)
    lo, hi, D = 0.9, 1.1, 6.0
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                     alpha=lo, beta=hi, guard_threshold=0.0, loss_denominator=D, variant="gspo")
    ht, Wt = torch.tensor(h, requires_grad=True), torch.tensor(W, requires_grad=True)
    lp = torch.log_softmax(ht @ Wt.T, 1)[torch.arange(b.T), torch.from_numpy(b.targets).long()]
    lm = torch.from_numpy(b.loss_mask.astype(bool))
    J = 0.0
    off = b.rollout_offsets
    for i in range(len(A)):
        sl = slice(int(off[i]), int(off[i + 1]))
        m = lm[sl]
        if m.sum() == 0:
            continue
        s = torch.exp(((lp[sl] - torch.from_numpy(infer[sl]))[m]).mean())
        J = J + torch.minimum(s * A[i], torch.clamp(s, lo, hi) * A[i])
    loss = -J / D
    loss.backward()
    assert loss.item() == pytest.approx(res.report.loss, abs=1e-13)
    np.testing.assert_allclose(res.d_hidden, ht.grad.numpy(), atol=1e-13)
    np.testing.assert_allclose(res.d_w_vocab, Wt.grad.numpy(), atol=1e-13)


def test_cispo_gradient_matches_torch_surrogate():
    """CISPO's gradient is that of sum sg(clip(k)) A logp / D (stop-gradient weight)."""
    b, h, W, infer = _tiny(5, dsig=0.8)
    A = oracle.group_advantages(b.rewards).reshape(-1)
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                     alpha=0.8, beta=1.2, guard_threshold=1e-5, variant="cispo")
    ht, Wt = torch.tensor(h, requires_grad=True), torch.tensor(W, requires_grad=True)
    lp = torch.log_softmax(ht @ Wt.T, 1)[torch.arange(b.T), torch.from_numpy(b.targets).long()]
    w = torch.from_numpy(res.report.coef)            # = keep * clip(k) * A / D, a constant
    loss = -(w * lp).sum()
    loss.backward()
    assert loss.item() == pytest.approx(res.report.loss, abs=1e-13)
    np.testing.assert_allclose(res.d_hidden, ht.grad.numpy(), atol=1e-13)
    np.testing.assert_allclose(res.d_w_vocab, Wt.grad.numpy(), atol=1e-13)
