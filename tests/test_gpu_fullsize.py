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


def _sampled_reference(b, rows, infer, adv, D, inv_temperature=1.0):
    """Oracle on a set of sampled rows (loss mask 1 only there): rollout structure
    re-based to the sampled rows, so the guard sees exactly the sampled tokens."""
    rollout_of = np.repeat(np.arange(len(b.rollout_offsets) - 1), np.diff(b.rollout_offsets))
    counts = np.bincount(rollout_of[rows], minlength=len(b.rollout_offsets) - 1)
    sub_off = np.concatenate([[0], np.cumsum(counts)])
    h64 = oracle.bf16_to_f64(b.hidden[rows])
    w64 = oracle.bf16_to_f64(b.w_vocab)
    return oracle.policy_loss_fwd_bwd(h64, w64, b.targets[rows], infer[rows].astype(np.float64), None, sub_off,
                                      None, loss_denominator=D, rollout_adv=adv.astype(np.float64),
                                      inv_temperature=inv_temperature)


def _sample_rows(b, n, seed):
    rows = np.sort(np.random.default_rng(seed).choice(b.T, size=n, replace=False))
    return rows


def _infer_for(b, rows):
    h64 = oracle.bf16_to_f64(b.hidden[rows])
    w64 = oracle.bf16_to_f64(b.w_vocab)
    lp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h64, w64), b.targets[rows])
    infer = np.full(b.T, -5.0, dtype=np.float32)
    infer[rows] = synth.compose_infer_logprobs(lp, b.delta_noise[rows] * 3.0, b.spikes[rows])
    return infer


def test_small_config_chunked_backward_sampled_rows():
    """BASELINE 'small dense' (T = 131072, H = 2048, V = 32000) with the bench's
    16k-row dU chunks (8 chunks; dW accumulated by TMA reduce-add)."""
    wl = synth.CONFIGS["small"]
    b = synth.make_batch(wl, 4)
    T, H, V = b.T, b.H, b.V
    rows = _sample_rows(b, 1536, 4)
    infer = _infer_for(b, rows)
    lm = np.zeros(T, np.uint8)
    lm[rows] = 1
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    D = float(len(rows))
    ref = _sampled_reference(b, rows, infer, adv, D)
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    hidden, w = bf(b.hidden), bf(b.w_vocab)
    tg = torch.from_numpy(b.targets).to(dev)
    shape = rl.make_shape(T, H, V)
    lp, ent, lse = (torch.empty(T, device=dev) for _ in range(3))
    ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, len(adv), 16384), dev)
    rl.rl_logprob_fwd(shape, hidden, w, tg, lp, ent, lse, workspace=ws)
    coef = torch.empty(T, device=dev)
    keep = torch.empty(T, dtype=torch.uint8, device=dev)
    guarded = torch.empty(len(adv), dtype=torch.uint8, device=dev)
    report = rl.new_report(dev)
    rl.rl_loss_coef(rl.make_params(len(adv), D), T, V, lp, torch.from_numpy(infer).to(dev), tg,
                    torch.from_numpy(adv).to(dev), torch.from_numpy(b.rollout_offsets).to(dev),
                    torch.from_numpy(lm).to(dev), coef, keep, guarded, report=report)
    dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(V, H, device=dev)
    rl.rl_bwd(shape, hidden, w, tg, lse, coef, d_hidden=dh, d_w_vocab=dw, dz_chunk_rows=16384, workspace=ws)
    torch.cuda.synchronize()
    assert np.max(np.abs(lp.cpu().numpy()[rows] - ref.logp)) <= harness.LOGP_TOL
    assert np.max(np.abs(ent.cpu().numpy()[rows] - ref.entropy)) <= harness.LOGP_TOL
    rep = rl.read_report(report).as_dict()
    assert abs(rep["loss"] - ref.report.loss) <= harness.LOSS_TOL
    assert harness.rel_fro(dh.float().cpu().numpy()[rows].astype(np.float64), ref.d_hidden) <= harness.GRAD_RTOL
    assert harness.rel_fro(dw.cpu().numpy().astype(np.float64), ref.d_w_vocab) <= harness.GRAD_RTOL


def test_glm64k_vocab_parallel_emulated_sampled_rows():
    """BASELINE 'GLM-4.5-Air long-context' (T = 65536, V = 151552) as 2 vocab
    shards through the split-phase ABI on one GPU (what each rank of the N = 2
    vocab-parallel run executes, in sequence), sampled rows checked vs the oracle."""
    wl = synth.CONFIGS["glm64k"]
    b = synth.make_batch(wl, 5)
    T, H, V = b.T, b.H, b.V
    rows = _sample_rows(b, 512, 5)
    infer = _infer_for(b, rows)
    lm = np.zeros(T, np.uint8)
    lm[rows] = 1
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    D = float(len(rows))
    ref = _sampled_reference(b, rows, infer, adv, D)
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    hidden = bf(b.hidden)
    tg = torch.from_numpy(b.targets).to(dev)
    n = 2
    Vl = V // n
    parts = torch.empty(n, T, 4, device=dev)
    shards = [bf(b.w_vocab[j * Vl:(j + 1) * Vl]) for j in range(n)]
    ws = None
    for j in range(n):
        shp = rl.make_shape(T, H, Vl, j * Vl, V)
        ws = ws if ws is not None else rl.alloc_workspace(rl.rl_workspace_bytes(shp, len(adv), 16384), dev)
        rl.rl_fwd_partials(shp, hidden, shards[j], tg, parts[j], workspace=ws)
    lp, ent, lse = (torch.empty(T, device=dev) for _ in range(3))
    rl.rl_merge_partials(parts, n, T, lp, ent, lse)
    coef = torch.empty(T, device=dev)
    report = rl.new_report(dev)
    rl.rl_loss_coef(rl.make_params(len(adv), D), T, V, lp, torch.from_numpy(infer).to(dev), tg,
                    torch.from_numpy(adv).to(dev), torch.from_numpy(b.rollout_offsets).to(dev),
                    torch.from_numpy(lm).to(dev), coef, report=report)
    dh = torch.zeros(T, H, device=dev)
    dws = []
    for j in range(n):
        shp = rl.make_shape(T, H, Vl, j * Vl, V)
        dhp = torch.empty(T, H, device=dev)
        dw = torch.empty(Vl, H, device=dev)
        rl.rl_bwd(shp, hidden, shards[j], tg, lse, coef, d_hidden_f32=dhp, d_w_vocab=dw, dz_chunk_rows=16384,
                  workspace=ws)
        dh += dhp
        dws.append(dw)
    torch.cuda.synchronize()
    assert np.max(np.abs(lp.cpu().numpy()[rows] - ref.logp)) <= harness.LOGP_TOL
    assert np.max(np.abs(ent.cpu().numpy()[rows] - ref.entropy)) <= harness.LOGP_TOL
    rep = rl.read_report(report).as_dict()
    assert abs(rep["loss"] - ref.report.loss) <= harness.LOSS_TOL
    assert harness.rel_fro(dh.cpu().numpy()[rows].astype(np.float64), ref.d_hidden) <= harness.GRAD_RTOL
    dw_all = torch.cat(dws).cpu().numpy().astype(np.float64)
    assert harness.rel_fro(dw_all, ref.d_w_vocab) <= harness.GRAD_RTOL


def test_stress_full_size_sparse_backward():
    """BASELINE 'stress' per rank (T = 16384, one G = 16 group, delta sigma 1.0,
    spikes 1e-4): every row is a loss row and ~43% of them are masked, so the
    sparse backward compacts thousands of rows over many tiles. The inference
    log-probs of all rows are the engine's own log-probs plus the stress noise.
    Checks: sampled rows' logprob/entropy vs the fp64 oracle; every coefficient
    equals the paper's gate recomputed on the host from the returned log-probs
    (Eq.2 closed interval, strict guard, A_i / D); dH of the sparse path is
    bitwise the dense path's and dW agrees to fp32 summation order; the masked
    rows' dH is exactly zero; sum_v dW[v, :] ~ 0."""
    wl = synth.Workload("stress-rank", 1, 16, 1024, 4096, 151552, delta_sigma=1.0, spike_rate=1e-4)
    b = synth.make_batch(wl, 7)
    T, H, V = b.T, b.H, b.V
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    hidden, w = bf(b.hidden), bf(b.w_vocab)
    targets = torch.from_numpy(b.targets).to(dev)
    shape = rl.make_shape(T, H, V)
    lp0 = torch.empty(T, device=dev)
    rl.rl_logprob_fwd(shape, hidden, w, targets, lp0)
    infer = synth.compose_infer_logprobs(lp0.cpu().numpy().astype(np.float64), b.delta_noise, b.spikes)
    adv = oracle.group_advantages(b.rewards).reshape(-1).astype(np.float32)
    D = float(T)
    params = rl.make_params(len(adv), D)
    off = b.rollout_offsets
    f32 = dict(dtype=torch.float32, device=dev)
    res = {}
    for dense in (False, True):
        out = dict(logprob=torch.empty(T, **f32), entropy=torch.empty(T, **f32), coef=torch.empty(T, **f32),
                   keep=torch.empty(T, dtype=torch.uint8, device=dev),
                   guarded=torch.empty(len(adv), dtype=torch.uint8, device=dev))
        report = rl.new_report(dev)
        dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        dw = torch.empty(V, H, **f32)
        rl.rl_policy_loss_fwd_bwd(shape, params, hidden, w, targets, torch.from_numpy(infer).to(dev),
                                  torch.from_numpy(adv).to(dev), torch.from_numpy(off).to(dev), None,
                                  report=report, logprob=out["logprob"], entropy=out["entropy"], coef=out["coef"],
                                  token_keep=out["keep"], rollout_guarded=out["guarded"], d_hidden=dh, d_w_vocab=dw,
                                  dense_backward=dense)
        torch.cuda.synchronize()
        res[dense] = ({k: v.cpu().numpy() for k, v in out.items()}, dh.view(torch.int16).cpu().numpy(),
                      dw.cpu().numpy(), rl.read_report(report, check=True))
    g, dh_s, dw_s, rep = res[False]
    _, dh_d, dw_d, _ = res[True]

    # sampled rows vs the fp64 oracle
    rows = _sample_rows(b, 512, 1)
    h64 = oracle.bf16_to_f64(b.hidden[rows])
    lp_ref, ent_ref, _ = oracle.log_softmax_stats(oracle.lm_logits(h64, oracle.bf16_to_f64(b.w_vocab)),
                                                   b.targets[rows])
    assert np.max(np.abs(g["logprob"][rows] - lp_ref)) <= harness.LOGP_TOL
    assert np.max(np.abs(g["entropy"][rows] - ent_ref)) <= harness.LOGP_TOL

    # the gate, recomputed from the returned log-probs (float64 on the host)
    k = np.exp(g["logprob"].astype(np.float64) - infer.astype(np.float64))
    rollout_of = np.repeat(np.arange(len(adv)), np.diff(off))
    kmin = np.full(len(adv), np.inf)
    np.minimum.at(kmin, rollout_of, k)
    guarded = kmin < synth.GUARD
    keep = (k >= synth.ALPHA) & (k <= synth.BETA) & ~guarded[rollout_of]
    near = (np.abs(k - synth.ALPHA) <= harness.BAND) | (np.abs(k - synth.BETA) <= harness.BAND)
    assert np.all(near[g["keep"].astype(bool) != keep])
    assert g["guarded"].astype(bool).tolist() == guarded.tolist()
    both = keep & g["keep"].astype(bool)
    coef_ref = k * adv[rollout_of] / D
    assert np.allclose(g["coef"][both], coef_ref[both], rtol=1e-4, atol=0)
    assert rep.masked_low + rep.masked_high > 0.2 * T       # heavy masking is exercised
    kept = g["coef"] != 0
    assert 0.3 * T < kept.sum() < 0.9 * T

    # sparse == dense backward; masked rows carry zero dH
    assert np.array_equal(dh_s, dh_d)
    assert not dh_s[~kept].any()
    assert harness.rel_fro(dw_s, dw_d) <= 1e-5
    col = np.linalg.norm(dw_s.astype(np.float64).sum(0)) / np.linalg.norm(dw_s.astype(np.float64))
    assert col < 1e-2
