"""Pins of the fp64 oracle against things other than itself (CPU, `-m "not gpu"`).

Each test names what fixes the expected value: a SPEC/paper example table, a
closed form, a library routine on a special case, finite differences, or an
invariant of the mathematics. A plausible slip in oracle/icepop.py (a dropped
term, a wrong sign or index, a transposed operand, an open instead of closed
interval, <= instead of <) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import oracle
import synth


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------ golden tables
def test_mask_ratio_spec_table(golden_dir):
    for c in _load(golden_dir, "spec_examples.json")["mask_ratio"]["cases"]:
        assert oracle.masking_function(np.array([c["k"]]), c["alpha"], c["beta"])[0] == c["out"]


def test_advantages_spec_table(golden_dir):
    for c in _load(golden_dir, "spec_examples.json")["advantages"]["cases"]:
        got = oracle.group_advantages(np.array([c["rewards"]], dtype=np.float64))[0]
        np.testing.assert_array_equal(got, np.array(c["out"], dtype=np.float64))


def test_advantages_reject_group_of_one():
    with pytest.raises(ValueError):
        oracle.group_advantages(np.array([[1.0]]))


def test_guard_spec_table(golden_dir):
    for c in _load(golden_dir, "spec_examples.json")["guard"]["cases"]:
        k = np.array(c["ratios"], dtype=np.float64)
        g = oracle.rollout_guard(k, np.array([0, len(k)]), np.ones(len(k), np.uint8), c["threshold"])
        assert bool(g[0]) == c["guarded"]


def test_hand_loss_example(golden_dir):
    ex = _load(golden_dir, "hand_loss_example.json")
    logp = np.array(ex["logp"])
    infer = logp - np.array(ex["log_ratio"])
    A = oracle.group_advantages(np.array(ex["rewards"], dtype=np.float64)).reshape(-1)
    rep = oracle.icepop_loss(logp, infer, A, np.array(ex["offsets"]), None, ex["alpha"],
                             ex["beta"], ex["guard"], ex["D"])
    assert rep.loss == pytest.approx(ex["loss"], abs=1e-14)
    np.testing.assert_allclose(rep.coef * ex["D"], ex["coef_times_D"], atol=1e-13)
    for key in ("masked_low", "masked_high", "guarded_rollouts", "guarded_tokens", "kept_tokens"):
        assert getattr(rep, key) == ex[key], key
    # k - ln k - 1 summed by hand over every valid token (catches a sum over kept tokens
    # only, a dropped -1, or ln k taken with the wrong sign)
    assert rep.mismatch_kl_sum == pytest.approx(ex["mismatch_kl_sum"], rel=1e-12)


# --------------------------------------------------------------- input decode
@pytest.mark.parametrize("bits,value", [
    (0x3F80, 1.0), (0xC000, -2.0), (0x3F81, 1.0 + 2.0 ** -7), (0x4049, 3.140625),
    (0x0001, 2.0 ** -133),                     # smallest subnormal: 2^-126 * 2^-7
    (0x0080, 2.0 ** -126),                     # smallest normal
    (0x7F7F, (2.0 - 2.0 ** -7) * 2.0 ** 127),  # largest finite
    (0x7F80, math.inf), (0xFF80, -math.inf),
])
def test_bf16_decode_known_bit_patterns(bits, value):
    """bf16 = the top 16 bits of an IEEE binary32 (sign, 8-bit exponent, 7-bit
    mantissa); each value above is worked out from that layout by hand. A wrong
    shift, a sign-extension of the uint16 or a float16 reinterpretation fails."""
    assert oracle.bf16_to_f64(np.array([bits], dtype=np.uint16))[0] == value


def test_bf16_decode_signed_zero_and_nan():
    z = oracle.bf16_to_f64(np.array([0x8000, 0x0000], dtype=np.uint16))
    assert z[0] == 0.0 and math.copysign(1.0, z[0]) == -1.0 and math.copysign(1.0, z[1]) == 1.0
    assert np.isnan(oracle.bf16_to_f64(np.array([0x7FC0, 0xFFC1], dtype=np.uint16))).all()


# ---------------------------------------------------------- closed forms
def test_uniform_logits_give_minus_log_v():
    """SPEC policy_logprobs: zero weights -> every log-prob is -ln V; entropy ln V."""
    T, H, V = 7, 16, 37
    h = np.random.default_rng(0).standard_normal((T, H))
    Z = oracle.lm_logits(h, np.zeros((V, H)))
    logp, ent, lse = oracle.log_softmax_stats(Z, np.arange(T) % V)
    np.testing.assert_allclose(logp, -math.log(V), rtol=0, atol=1e-14)
    np.testing.assert_allclose(ent, math.log(V), rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse, math.log(V), rtol=0, atol=1e-14)


def test_two_level_logits_closed_form():
    """k entries at a, V-k at b: lse = log(k e^a + (V-k) e^b), p_a = e^a / (k e^a + (V-k) e^b),
    entropy = -k p_a log p_a - (V-k) p_b log p_b."""
    V, k, a, b = 50, 3, 7.25, -1.5
    z = np.full((1, V), b)
    z[0, [4, 11, 40]] = a
    den = k * math.exp(a) + (V - k) * math.exp(b)
    pa, pb = math.exp(a) / den, math.exp(b) / den
    logp, ent, lse = oracle.log_softmax_stats(z, np.array([11]))
    assert lse[0] == pytest.approx(math.log(den), abs=1e-13)
    assert logp[0] == pytest.approx(math.log(pa), abs=1e-13)
    assert ent[0] == pytest.approx(-k * pa * math.log(pa) - (V - k) * pb * math.log(pb), abs=1e-13)


def test_logits_are_the_scaled_product():
    """z[t, v] = invT * <h_t, W_v>: checked entry-by-entry with math.fsum (no BLAS)."""
    rng = np.random.default_rng(1)
    h, W = rng.standard_normal((5, 9)), rng.standard_normal((13, 9))
    Z = oracle.lm_logits(h, W, 1 / 0.7, vocab_block=4)
    for t in range(5):
        for v in range(13):
            assert Z[t, v] == pytest.approx(math.fsum(h[t] * W[v]) / 0.7, rel=1e-13, abs=1e-13)


def test_normalisation_and_library_log_softmax():
    """sum_v exp(logp_v) = 1 (SPEC policy_logprobs example 3) and agreement with
    scipy.special.logsumexp / torch.log_softmax(float64) (library special case)."""
    rng = np.random.default_rng(2)
    Z = rng.standard_normal((6, 300)) * 5
    for t in range(6):
        logp_all = np.array([oracle.log_softmax_stats(Z[t:t + 1], np.array([v]))[0][0]
                             for v in range(300)])
        assert abs(np.exp(logp_all).sum() - 1.0) < 1e-12
        ref = torch.log_softmax(torch.from_numpy(Z[t]), dim=0).numpy()
        np.testing.assert_allclose(logp_all, ref, atol=1e-12)
    _, ent, lse = oracle.log_softmax_stats(Z, np.zeros(6, np.int64))
    np.testing.assert_allclose(lse, scipy.special.logsumexp(Z, axis=1), atol=1e-12)
    P = scipy.special.softmax(Z, axis=1)
    np.testing.assert_allclose(ent, -(P * np.log(P)).sum(axis=1), atol=1e-11)


# ----------------------------------------------------------- loss semantics
def _tiny_step(seed=0, T=None, mask_frac=0.0, invT=1.0, delta_sigma=0.3):
    wl = synth.Workload("t", 2, 3, 8, 8, 16, delta_sigma=delta_sigma, prompt_frac=mask_frac,
                        ragged=True, sigma_z=2.0)
    b = synth.make_batch(wl, seed)
    h, W = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h, W, invT)
    logp, _, _ = oracle.log_softmax_stats(Z, b.targets)
    infer = synth.compose_infer_logprobs(logp, b.delta_noise, b.spikes).astype(np.float64)
    return b, h, W, infer


def test_on_policy_closed_form():
    """SPEC invariant: train == infer gives k = 1, nothing masked, and
    loss = -(1/D) sum_i |y_i| A_i; zero when the rollouts of a group are equally long."""
    b, h, W, _ = _tiny_step()
    Z = oracle.lm_logits(h, W)
    logp, _, _ = oracle.log_softmax_stats(Z, b.targets)
    A = oracle.group_advantages(b.rewards).reshape(-1)
    off = b.rollout_offsets
    D = b.loss_denominator
    rep = oracle.icepop_loss(logp, logp, A, off, None, 0.5, 5.0, 1e-5, D)
    np.testing.assert_allclose(rep.ratio, 1.0, atol=1e-12)
    assert rep.kept_tokens == b.T and rep.masked_low == rep.masked_high == rep.guarded_rollouts == 0
    lens = np.diff(off)
    assert rep.loss == pytest.approx(-(lens * A).sum() / D, abs=1e-14)
    eq = np.full(len(A), 4)
    off_eq = np.concatenate([[0], np.cumsum(eq)])
    rep2 = oracle.icepop_loss(np.zeros(off_eq[-1]), np.zeros(off_eq[-1]), A, off_eq, None,
                              0.5, 5.0, 1e-5, float(off_eq[-1]))
    assert abs(rep2.loss) < 1e-15


def test_mask_is_hard_zero_and_denominator_counts_masked():
    """A token with k=6 contributes exactly 0 (SPEC icepop_loss example 2); the
    denominator is the caller's D, not the kept count (reading R5)."""
    logp = np.log(np.array([6.0, 1.0]))
    rep = oracle.icepop_loss(logp, np.zeros(2), np.array([1.0]), np.array([0, 2]), None,
                             0.5, 5.0, 1e-5, 2.0)
    assert rep.coef[0] == 0.0 and rep.keep.tolist() == [False, True]
    assert rep.loss == pytest.approx(-0.5, abs=1e-15)


def test_guard_uses_loss_tokens_only_and_counts():
    """Guard ignores loss_mask=0 tokens (reading R4); invalid infer values are
    excluded and counted."""
    logp = np.array([-20.0, -1.0, -1.0, -1.0])
    infer = np.array([0.0, -1.0, np.nan, 0.5])
    lm = np.array([0, 1, 1, 1], np.uint8)
    rep = oracle.icepop_loss(logp, infer, np.array([1.0]), np.array([0, 4]), lm, 0.5, 5.0, 1e-5, 3.0)
    assert rep.guarded_rollouts == 0 and rep.kept_tokens == 1 and rep.nonfinite_inputs == 2
    lm2 = np.array([1, 1, 1, 1], np.uint8)
    rep2 = oracle.icepop_loss(logp, infer, np.array([1.0]), np.array([0, 4]), lm2, 0.5, 5.0, 1e-5, 3.0)
    assert rep2.guarded_rollouts == 1 and rep2.kept_tokens == 0 and rep2.guarded_tokens == 2


def test_bad_offsets_neutralise_batch():
    rep = oracle.icepop_loss(np.zeros(4), np.zeros(4), np.array([1.0, 1.0]), np.array([0, 3, 2]),
                             None, 0.5, 5.0, 1e-5, 4.0)
    assert rep.bad_offsets == 1 and rep.loss == 0.0 and not rep.keep.any()


def test_advantage_zero_sum_and_linearity():
    rng = np.random.default_rng(3)
    S = rng.random((10000, 16))
    A = oracle.group_advantages(S)
    assert np.abs(A.sum(axis=1)).max() < 1e-12
    np.testing.assert_allclose(oracle.group_advantages(3.5 * S), 3.5 * A, atol=1e-13)


# --------------------------------------------------------------- gradients
def _loss_of(h, W, b, infer, A, keep_fixed, invT):
    """loss(h, W) with the gate `keep_fixed` held constant (hard mask)."""
    Z = oracle.lm_logits(h, W, invT)
    logp, _, _ = oracle.log_softmax_stats(Z, b.targets)
    rollout_of = np.repeat(np.arange(len(A)), np.diff(b.rollout_offsets))
    return -(np.where(keep_fixed, np.exp(logp - infer) * A[rollout_of], 0.0)).sum() / b.loss_denominator


@pytest.mark.parametrize("seed", range(6))
def test_gradient_finite_differences(seed):
    """Central differences, step 1e-6, fp64 (SPEC icepop_gradient example 3);
    instances whose ratios sit within 1e-3 of alpha, beta or the guard are skipped."""
    invT = 1.0 if seed % 2 == 0 else 1 / 0.7
    b, h, W, infer = _tiny_step(seed, mask_frac=0.25 if seed % 3 == 0 else 0.0, invT=invT,
                                delta_sigma=0.8)
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets,
                                     b.loss_mask, inv_temperature=invT)
    k = res.report.ratio
    for bound in (0.5, 5.0):
        if np.any(np.abs(k - bound) < 1e-3):
            pytest.skip("ratio within 1e-3 of a mask bound")
    keep = res.report.keep
    A = res.advantages
    eps = 1e-6
    rng = np.random.default_rng(seed)
    for (X, G) in ((h, res.d_hidden), (W, res.d_w_vocab)):
        idx = [tuple(rng.integers(0, s) for s in X.shape) for _ in range(25)]
        num, ana = [], []
        for ix in idx:
            old = X[ix]
            X[ix] = old + eps
            lp = _loss_of(h, W, b, infer, A, keep, invT)
            X[ix] = old - eps
            lm_ = _loss_of(h, W, b, infer, A, keep, invT)
            X[ix] = old
            num.append((lp - lm_) / (2 * eps))
            ana.append(G[ix])
        num, ana = np.array(num), np.array(ana)
        assert np.linalg.norm(num - ana) <= 1e-5 * max(np.linalg.norm(ana), 1e-12)


def test_gradient_matches_torch_autograd():
    """Library special case: torch float64 autograd of -(1/D) sum keep k A."""
    b, h, W, infer = _tiny_step(4, delta_sigma=0.8)
    invT = 1 / 0.7
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets,
                                     inv_temperature=invT)
    ht = torch.tensor(h, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    lp = torch.log_softmax((ht @ Wt.T) * invT, dim=1)[torch.arange(b.T), torch.from_numpy(b.targets).long()]
    rollout_of = np.repeat(np.arange(len(res.advantages)), np.diff(b.rollout_offsets))
    A_tok = torch.from_numpy(res.advantages[rollout_of])
    keep = torch.from_numpy(res.report.keep)
    loss = -(torch.where(keep, torch.exp(lp - torch.from_numpy(infer)) * A_tok,
                         torch.zeros(()).double())).sum() / b.loss_denominator
    loss.backward()
    assert loss.item() == pytest.approx(res.report.loss, abs=1e-14)
    np.testing.assert_allclose(res.d_hidden, ht.grad.numpy(), atol=1e-14)
    np.testing.assert_allclose(res.d_w_vocab, Wt.grad.numpy(), atol=1e-14)


def test_gradient_invariants():
    """sum_v dZ_tv = 0 => sum_v dW[v,:] = 0; dH_t = invT coef_t (E_p[W] - W_y)."""
    b, h, W, infer = _tiny_step(5, delta_sigma=0.5)
    invT = 1.3
    res = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets,
                                     inv_temperature=invT)
    assert np.abs(res.d_w_vocab.sum(axis=0)).max() < 1e-14
    Z = oracle.lm_logits(h, W, invT)
    P = scipy.special.softmax(Z, axis=1)
    ref = invT * res.report.coef[:, None] * (P @ W - W[b.targets])
    np.testing.assert_allclose(res.d_hidden, ref, atol=1e-14)


def test_zero_advantage_or_all_masked_gives_zero_gradient():
    b, h, W, infer = _tiny_step(6)
    r0 = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, np.ones_like(b.rewards),
                                    b.rollout_offsets)
    assert not r0.d_hidden.any() and not r0.d_w_vocab.any()
    r1 = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets,
                                    alpha=10.0, beta=20.0)
    assert r1.report.loss == 0.0 and not r1.d_hidden.any() and not r1.d_w_vocab.any()


# ---------------------------------------------------------- shard identity
def test_vocab_shard_merge_identity():
    """Splitting the vocab into shards and merging (m, s, t, z_target) reproduces
    the unsharded lse, entropy and target logit (associativity of the merge)."""
    rng = np.random.default_rng(7)
    Z = rng.standard_normal((9, 103)) * 4
    y = rng.integers(0, 103, 9)
    logp, ent, lse = oracle.log_softmax_stats(Z, y)
    cuts = [0, 10, 50, 51, 103]
    parts = [oracle.shard_stats(Z[:, a:b], y, a) for a, b in zip(cuts[:-1], cuts[1:])]
    lse2, ent2, zt = oracle.merge_shard_stats(parts)
    np.testing.assert_allclose(lse2, lse, atol=1e-13)
    np.testing.assert_allclose(ent2, ent, atol=1e-12)
    np.testing.assert_allclose(zt - lse2, logp, atol=1e-13)


def test_oracle_deterministic():
    b, h, W, infer = _tiny_step(8)
    r1 = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets)
    r2 = oracle.policy_loss_fwd_bwd(h, W, b.targets, infer, b.rewards, b.rollout_offsets)
    assert r1.report.loss == r2.report.loss
    assert np.array_equal(r1.d_w_vocab, r2.d_w_vocab)


# ------------------------------------------------- direct pins of the remaining helpers
def test_validate_offsets_hand_cases():
    """CSR rollout offsets (SPEC 'misaligned lengths'): start at 0, end at T,
    never decrease. Each rule broken once."""
    from oracle.icepop import validate_offsets
    assert validate_offsets([0, 3, 3, 7], 7)            # an empty rollout is fine
    assert validate_offsets([0], 0)
    assert not validate_offsets([1, 3, 7], 7)           # does not start at 0
    assert not validate_offsets([0, 3, 6], 7)           # does not end at T
    assert not validate_offsets([0, 5, 3, 7], 7)        # decreasing


def test_icepop_backward_hand_example():
    """dZ = coef invT (softmax - onehot), dH = dZ W, dW = dZ^T h on a 1-row, 2-word
    vocabulary worked by hand: z = (0, ln 3) -> p = (1/4, 3/4); y = 1, coef = 2,
    invT = 1/2 -> dZ = 2 * 1/2 * (1/4, 3/4 - 1) = (1/4, -1/4)."""
    Z = np.array([[0.0, np.log(3.0)]])
    lse = np.array([np.log(4.0)])
    h = np.array([[2.0, -1.0]])
    W = np.array([[1.0, 0.0], [0.0, 1.0]])
    dZ, dH, dW = oracle.icepop_backward(Z, lse, np.array([1]), np.array([2.0]), h, W, 0.5)
    np.testing.assert_allclose(dZ, [[0.25, -0.25]], atol=1e-15)
    np.testing.assert_allclose(dH, [[0.25, -0.25]], atol=1e-15)          # dZ @ I
    np.testing.assert_allclose(dW, [[0.5, -0.25], [-0.5, 0.25]], atol=1e-15)   # dZ^T h


def test_variant_loss_dispatch():
    """variant_loss is a name -> function table: each name reaches its own definition
    (a swapped entry would compute another variant's coefficients)."""
    from oracle import icepop as ic
    rng = np.random.default_rng(4)
    lp = -rng.uniform(0.1, 3.0, 12)
    inf = lp + rng.normal(0, 0.5, 12)
    inf = np.minimum(inf, 0.0)
    args = (lp, inf, np.array([0.5, -0.5, 1.0]), np.array([0, 4, 8, 12]), None, 0.8, 1.2, 1e-5, 12.0)
    for name, fn in (("icepop", ic.icepop_loss), ("cispo", ic.cispo_loss), ("gspo", ic.gspo_loss)):
        a, b = ic.variant_loss(name, *args), fn(*args)
        np.testing.assert_array_equal(a.coef, b.coef)
        assert a.loss == b.loss
    assert not np.array_equal(ic.variant_loss("icepop", *args).coef, ic.variant_loss("cispo", *args).coef)


def test_grouped_mm_rmsnorm_hand_example():
    """The expert projection of normalised tokens on a 1-token, 1-expert case by hand:
    x = (3, 4) -> rms = sqrt(12.5), gamma = (1, 2), W = [[1, 1]] ->
    y = (3 * 1 + 4 * 2) / sqrt(12.5) = 11 / sqrt(12.5)."""
    from oracle import moe
    y = moe.grouped_mm_rmsnorm(np.array([[3.0, 4.0]]), np.array([1.0, 2.0]), np.array([[[1.0, 1.0]]]),
                               np.array([0, 1]), eps=0.0)
    assert y[0, 0] == pytest.approx(11.0 / np.sqrt(12.5), rel=1e-14)
