"""Pins for the oracle's KL term (reading R19) and per-token temperature (R20), the
remaining SURVEY §8 f2 items. Neither is in PAPER.md's Eq.1 (defaults: kl_tau = 0,
one scalar temperature), so they are pinned against mathematics, not the paper:
central differences of the objective they define, the on-policy closed form, the
identity at kl_tau = 0 / constant temperatures, and a scale invariance."""
import numpy as np
import pytest

import oracle
import synth


def _tiny(seed, invT=1.0, dsig=0.8, mask_frac=0.25):
    wl = synth.Workload("t", 2, 3, 8, 8, 16, delta_sigma=dsig, prompt_frac=mask_frac, ragged=True, sigma_z=2.0)
    b = synth.make_batch(wl, seed)
    h, W = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h, W, invT)
    logp, _, _ = oracle.log_softmax_stats(Z, b.targets)
    infer = synth.compose_infer_logprobs(logp, b.delta_noise, b.spikes).astype(np.float64)
    return b, h, W, infer


def _objective(h, W, b, infer, A, keep, S, kl_tau, invT):
    """-(1/D) sum keep k A + (kl_tau/D) sum_S log k, gates held fixed (R2, R19)."""
    logp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h, W, invT), b.targets)
    rollout_of = np.repeat(np.arange(len(A)), np.diff(b.rollout_offsets))
    D = b.loss_denominator
    pg = -(np.where(keep, np.exp(logp - infer) * A[rollout_of], 0.0)).sum() / D
    return pg + kl_tau / D * np.where(S, logp - infer, 0.0).sum()


def _fd_check(h, W, grads, f, seed, n=20, eps=1e-6):
    rng = np.random.default_rng(seed)
    for X, G in ((h, grads[0]), (W, grads[1])):
        num, ana = [], []
        for _ in range(n):
            ix = tuple(rng.integers(0, s) for s in X.shape)
            old = X[ix]
            X[ix] = old + eps
            fp = f()
            X[ix] = old - eps
            fm = f()
            X[ix] = old
            num.append((fp - fm) / (2 * eps))
            ana.append(G[ix])
        num, ana = np.array(num), np.array(ana)
        assert np.linalg.norm(num - ana) <= 1e-5 * max(np.linalg.norm(ana), 1e-12)


@pytest.mark.parametrize("kl_set", ["masked", "unmasked", "all"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_kl_term_finite_differences(kl_set, seed):
    b, h, W, infer = _tiny(seed)
    kl_tau = 0.37
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                     kl_tau=kl_tau, kl_set=kl_set)
    k = res.report.ratio
    if np.any(np.abs(k - 0.5) < 1e-3) or np.any(np.abs(k - 5.0) < 1e-3):
        pytest.skip("ratio within 1e-3 of a mask bound")
    rep = res.report
    S = {"masked": rep.valid & ~rep.keep, "unmasked": rep.keep, "all": rep.valid}[kl_set]
    assert S.any()
    # the reported loss is the objective's value
    assert res.report.loss == pytest.approx(_objective(h, W, b, infer, res.advantages, rep.keep, S, kl_tau, 1.0),
                                            abs=1e-14)
    _fd_check(h, W, (res.d_hidden, res.d_w_vocab),
              lambda: _objective(h, W, b, infer, res.advantages, rep.keep, S, kl_tau, 1.0), seed)


def test_kl_term_on_policy_closed_form_and_identity():
    """infer := logp gives log k = 0: the loss is the kl_tau = 0 loss and every coef
    on the KL set is shifted by exactly -kl_tau / D; kl_tau = 0 is the identity."""
    b, h, W, _ = _tiny(3, mask_frac=0.25)
    logp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h, W), b.targets)
    A = oracle.group_advantages(b.rewards).reshape(-1)
    D = b.loss_denominator
    base = oracle.icepop_loss(logp, logp, A, b.rollout_offsets, b.loss_mask, 0.5, 5.0, 1e-5, D)
    for kl_set in oracle.KL_SETS:
        r = oracle.add_kl_term(base, logp, logp, 0.25, kl_set, D)
        assert r.loss == base.loss
        S = {"masked": base.valid & ~base.keep, "unmasked": base.keep, "all": base.valid}[kl_set]
        np.testing.assert_array_equal(r.coef, base.coef - np.where(S, 0.25 / D, 0.0))
    assert oracle.add_kl_term(base, logp, logp + 0.3, 0.0, "all", D) is base


def test_kl_term_hand_example():
    """Two rollouts, hand values: S = masked tokens (one low, one guarded rollout)."""
    logp = np.log(np.array([1.0, 0.4, 2.0, 1e-6, 1.0]))   # with infer = 0: k = exp(logp)
    infer = np.zeros(5)
    off = np.array([0, 3, 5])
    A = np.array([0.5, -0.5])
    rep = oracle.icepop_loss(logp, infer, A, off, None, 0.5, 5.0, 1e-5, 5.0)
    # rollout 0: k = 1, 0.4 (< alpha: masked), 2 -> kept {0, 2}; rollout 1 guarded (1e-6 < 1e-5)
    assert rep.keep.tolist() == [True, False, True, False, False]
    r = oracle.add_kl_term(rep, logp, infer, 2.0, "masked", 5.0)
    S_logk = np.log(0.4) + np.log(1e-6) + np.log(1.0)
    assert r.loss == pytest.approx(-(1.0 * 0.5 + 2.0 * 0.5) / 5.0 + 2.0 / 5.0 * S_logk, abs=1e-15)


def test_per_token_temperature_constant_equals_scalar():
    b, h, W, infer = _tiny(4, invT=1 / 0.7)
    a = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                   inv_temperature=1 / 0.7)
    c = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                   inv_temperature=np.full(b.T, 1 / 0.7))
    for x, y in ((a.logp, c.logp), (a.entropy, c.entropy), (a.report.coef, c.report.coef),
                 (a.d_hidden, c.d_hidden), (a.d_w_vocab, c.d_w_vocab)):
        np.testing.assert_array_equal(x, y)


def test_per_token_temperature_scale_invariance():
    """z_t = invT_t h_t W^T: (c_t h_t, invT_t / c_t) gives the same logits, so the
    same logp, and dH_t scales by 1 / c_t."""
    b, h, W, infer = _tiny(5)
    rng = np.random.default_rng(0)
    invT = rng.uniform(0.5, 2.0, b.T)
    c = 2.0 ** rng.integers(-2, 3, b.T)                     # powers of two: exact rescaling
    a = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                   inv_temperature=invT)
    s = oracle.policy_loss_fwd_bwd(h * c[:, None], W, b.targets, infer, b.rewards, b.rollout_offsets,
                                   b.loss_mask, inv_temperature=invT / c)
    np.testing.assert_allclose(s.logp, a.logp, rtol=0, atol=1e-13)
    np.testing.assert_allclose(s.d_hidden * c[:, None], a.d_hidden, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(s.d_w_vocab, a.d_w_vocab, rtol=1e-11, atol=1e-15)


@pytest.mark.parametrize("seed", [6, 7])
def test_per_token_temperature_finite_differences(seed):
    b, h, W, infer = _tiny(seed)
    invT = np.random.default_rng(seed).uniform(0.6, 1.7, b.T)
    infer = synth.compose_infer_logprobs(
        oracle.log_softmax_stats(oracle.lm_logits(h, W, invT), b.targets)[0], b.delta_noise, b.spikes)
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask,
                                     inv_temperature=invT, kl_tau=0.2, kl_set="all")
    k = res.report.ratio
    if np.any(np.abs(k - 0.5) < 1e-3) or np.any(np.abs(k - 5.0) < 1e-3):
        pytest.skip("ratio within 1e-3 of a mask bound")
    rep = res.report
    _fd_check(h, W, (res.d_hidden, res.d_w_vocab),
              lambda: _objective(h, W, b, infer, res.advantages, rep.keep, rep.valid, 0.2, invT), seed)
