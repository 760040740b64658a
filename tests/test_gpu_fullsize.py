"""Parity at BASELINE.json's full GLM-4.5-Air shape (T = 16384, H = 4096,
V = 151552) in the launch configuration bench.py times (`-m gpu`).

The fp64 oracle cannot afford the whole 16k x 151552 x 4096 forward, so the
batch's loss mask is zero outside two sampled rollouts (2048 rows). The CUDA path
still runs every kernel at full size; every output it produces is then something
the oracle can compute from the sampled rows alone:
  * logprob / entropy / lse of the sampled rows (each row is independent);
  * Eq.1/Eq.2/guard coefficients, keep flags and the loss of the sampled rollouts;
  * dH of the sampled rows, and the WHOLE dW, since coef = 0 elsewhere.
Other rows' logprob/entropy are checked against properties that hold at any size
(entropy in [0, ln V], logprob <= 0, finite)."""
import math

import numpy as np
import pytest

import harness
import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402


def test_glm16k_sampled_rollouts():
    wl = synth.CONFIGS["glm16k"]
    b = synth.make_batch(wl, 3)
    T, H, V = b.T, b.H, b.V
    off = b.rollout_offsets
    sample = [5, 11]                                   # two whole rollouts
    rows = np.concatenate([np.arange(off[i], off[i + 1]) for i in sample])
    h64 = oracle.bf16_to_f64(b.hidden[rows])
    w64 = oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h64, w64)
    lp_ref, _, _ = oracle.log_softmax_stats(Z, b.targets[rows])
    del Z
    infer = np.full(T, -5.0, dtype=np.float32)
    spikes = b.spikes.copy()
    spikes[rows[100]] = True                          # force a guard spike in the first sampled rollout
    infer[rows] = synth.compose_infer_logprobs(lp_ref, b.delta_noise[rows], spikes[rows])
    lm = np.zeros(T, dtype=np.uint8)
    lm[rows] = 1
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    D = float(len(rows))

    # oracle on the sampled rollouts only (coef is zero everywhere else)
    sub_off = np.array([0, off[sample[0] + 1] - off[sample[0]], len(rows)], dtype=np.int64)
    ref = oracle.policy_loss_fwd_bwd(h64, w64, b.targets[rows], infer[rows].astype(np.float64), None, sub_off,
                                     None, loss_denominator=D, rollout_adv=adv[sample].astype(np.float64))
    assert ref.report.guarded_rollouts == 1

    # CUDA path at full size
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    hidden, w = bf(b.hidden), bf(b.w_vocab)
    f32 = dict(dtype=torch.float32, device=dev)
    out = dict(logprob=torch.empty(T, **f32), entropy=torch.empty(T, **f32), lse=torch.empty(T, **f32),
               coef=torch.empty(T, **f32), keep=torch.empty(T, dtype=torch.uint8, device=dev),
               guarded=torch.empty(len(adv), dtype=torch.uint8, device=dev))
    report = rl.new_report(dev)
    dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(V, H, **f32)
    shape = rl.make_shape(T, H, V)
    params = rl.make_params(len(adv), D)
    rl.rl_policy_loss_fwd_bwd(shape, params, hidden, w, torch.from_numpy(b.targets).to(dev),
                              torch.from_numpy(infer).to(dev), torch.from_numpy(adv).to(dev),
                              torch.from_numpy(off).to(dev), torch.from_numpy(lm).to(dev), report=report,
                              logprob=out["logprob"], entropy=out["entropy"], lse=out["lse"], coef=out["coef"],
                              token_keep=out["keep"], rollout_guarded=out["guarded"], d_hidden=dh, d_w_vocab=dw)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    rep = rl.read_report(report).as_dict()

    assert np.max(np.abs(g["logprob"][rows] - ref.logp)) <= harness.LOGP_TOL
    assert np.max(np.abs(g["entropy"][rows] - ref.entropy)) <= harness.LOGP_TOL
    assert np.max(np.abs(g["lse"][rows] - ref.lse)) <= harness.LOGP_TOL
    # any-size properties on every row
    assert np.all(np.isfinite(g["logprob"])) and np.all(g["logprob"] <= 1e-4)
    assert np.all(g["entropy"] >= -1e-4) and np.all(g["entropy"] <= math.log(V) + 1e-4)
    # S3 on the sampled rollouts, at the mask-band reading R13
    band = harness.band_tokens(harness.Case(None, None, None, None, None, 1.0), ref)
    flips = np.nonzero(g["keep"][rows].astype(bool) != ref.report.keep)[0]
    assert np.all(band[flips])
    assert g["guarded"][sample].astype(bool).tolist() == ref.report.guarded.tolist()
    assert not np.any(g["coef"][np.setdiff1d(np.arange(T), rows)])
    assert abs(rep["loss"] - ref.report.loss) <= harness.LOSS_TOL
    assert abs(rep["kept_tokens"] - ref.report.kept_tokens) <= int(band.sum())
    # gradients: dH rows and the whole dW
    assert harness.rel_fro(dh.float().cpu().numpy()[rows].astype(np.float64), ref.d_hidden) <= harness.GRAD_RTOL
    other = np.setdiff1d(np.arange(T), rows)[::97]
    assert not dh[torch.from_numpy(other).to(dev)].float().abs().max().item()
    dw_h = dw.cpu().numpy().astype(np.float64)
    assert harness.rel_fro(dw_h, ref.d_w_vocab) <= harness.GRAD_RTOL
