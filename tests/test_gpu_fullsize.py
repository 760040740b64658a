"""Parity at BASELINE.json's full sizes (`-m gpu`).

GLM-4.5-Air shape (T = 16384, H = 4096, V = 151552) in the launch configuration
bench.py times, EVERY row a loss row, sparse and dense backward: the fp64 oracle
runs one chunked pass over all 16384 rows (logits of 1024 rows at a time), which
gives lse / logprob / entropy of every row, the rollouts' sampled targets (the
policy's own samples), the whole Eq.1/Eq.2/guard gate, and the
terms the gradient needs on a sample: E_p[W] of >= 4096 rows (dH is per row) and
p[:, v] of 2 vocab rows per 256-row dW tile plus target rows (dW rows are sums over
all t). Band-edge tokens are planted at ln alpha, ln beta, ln tau_g +- {1e-6, 2e-4,
1e-3}. Two workloads: glm16k (delta sigma 0.3) and the per-rank stress batch (delta
sigma 1.0, ~40% of rows masked, so the sparse backward compacts many tiles).

The small / glm64k configs are checked on sampled rows (loss mask 1 there only).
"""
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




# ------------------------------------------------------------ all rows, full size
def _oracle_pass(b, h64, w64, dh_rows, dw_rows, chunk=1024):
    """One chunked fp64 oracle pass over every row: per row lse / entropy (target-free),
    the sampled target and the logit at it, the least likely token (guard spikes and
    plants) and its logit; E_p[W] for the dH sample rows; p[:, dw_rows] for all rows."""
    T, V = b.T, b.V
    out = dict(lse=np.empty(T), entropy=np.empty(T), targets=np.empty(T, np.int32), z_y=np.empty(T),
               amin=np.empty(T, np.int64), z_min=np.empty(T), E=np.empty((len(dh_rows), w64.shape[1])),
               PS=np.empty((T, len(dw_rows))))
    pos = {int(r): i for i, r in enumerate(dh_rows)}
    for c0 in range(0, T, chunk):
        c1 = min(T, c0 + chunk)
        Z = oracle.lm_logits(h64[c0:c1], w64)
        _, ent, lse = oracle.log_softmax_stats(Z, np.zeros(c1 - c0, np.int64))
        y = harness.sample_from_policy(Z, lse, b.sample_u[c0:c1])
        rows = np.arange(c1 - c0)
        amin = np.argmin(Z, axis=1)
        y = np.where(b.spikes[c0:c1], amin, y).astype(np.int32)   # guard spikes: the least likely token
        out["lse"][c0:c1], out["entropy"][c0:c1], out["targets"][c0:c1] = lse, ent, y
        out["z_y"][c0:c1], out["amin"][c0:c1], out["z_min"][c0:c1] = Z[rows, y], amin, Z[rows, amin]
        sel = [r - c0 for r in dh_rows if c0 <= r < c1]
        if sel:
            P = np.exp(Z[sel] - lse[sel, None])
            out["E"][[pos[r + c0] for r in sel]] = P @ w64
        out["PS"][c0:c1] = np.exp(Z[:, dw_rows] - lse[:, None])
        del Z
    return out


class _Ref:
    """What harness.compare reads from an oracle result (no full-size gradients)."""

    def __init__(self, logp, entropy, lse, report):
        self.logp, self.entropy, self.lse, self.report = logp, entropy, lse, report


def _gpu_step(c, dense):
    """The whole step at full size through the C ABI (K0 from the rewards), as the bench
    launches it (one 16384-row dU chunk). Returns host copies of everything compared."""
    b = c.batch
    dev = "cuda"
    d = harness.to_device(c, dev)
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    adv = rl.rl_group_advantages(d["rewards"], b.rewards.shape[1])
    f32 = dict(dtype=torch.float32, device=dev)
    out = dict(logprob=torch.empty(T, **f32), entropy=torch.empty(T, **f32), lse=torch.empty(T, **f32),
               coef=torch.empty(T, **f32), keep=torch.empty(T, dtype=torch.uint8, device=dev),
               guarded=torch.empty(R, dtype=torch.uint8, device=dev))
    report = rl.new_report(dev)
    dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(V, H, **f32)
    rl.rl_policy_loss_fwd_bwd(rl.make_shape(T, H, V), rl.make_params(R, b.loss_denominator), d["hidden"], d["w"],
                              d["targets"], d["infer"], adv, d["offsets"], d["loss_mask"], report=report,
                              logprob=out["logprob"], entropy=out["entropy"], lse=out["lse"], coef=out["coef"],
                              token_keep=out["keep"], rollout_guarded=out["guarded"], d_hidden=dh, d_w_vocab=dw,
                              dz_chunk_rows=T, dense_backward=dense)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    g["report"] = rl.read_report(report, check=True).as_dict()
    g["dh"] = dh.float().cpu().numpy().astype(np.float64)
    g["dw_colsum"] = float(dw.double().sum(0).norm() / dw.double().norm())
    return g, dw


FULL = {
    "glm16k": synth.CONFIGS["glm16k"],
    "stress": synth.Workload("stress-rank", 1, 16, 1024, 4096, 151552, delta_sigma=1.0, spike_rate=1e-4),
}


@pytest.mark.parametrize("name", list(FULL))
def test_full_size_all_rows_vs_oracle(name):
    wl = FULL[name]
    b = synth.make_batch(wl, 3)
    T, H, V = b.T, b.H, b.V
    if name == "glm16k":   # the bytes are the committed ones (tests/golden/generator_glm16k_seed3.json)
        import json
        import os
        from synth import artifact
        gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "generator_glm16k_seed3.json")))
        d = artifact.digests(artifact.batch_arrays(b, np.zeros(T, np.float32)))
        assert {k: d[k] for k in gold["sha256"]} == gold["sha256"]
    rng = np.random.default_rng(1234)
    dh_rows = np.sort(rng.choice(T, size=4096, replace=False))
    blocks = np.arange(0, V, 256)
    dw_rows = np.unique(np.concatenate([blocks + rng.integers(0, 256, size=len(blocks)),
                                        blocks + rng.integers(0, 256, size=len(blocks))]))
    dw_rows = dw_rows[dw_rows < V]
    h64, w64 = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    o = _oracle_pass(b, h64, w64, dh_rows, dw_rows)
    b.targets = o["targets"]
    logp = o["z_y"] - o["lse"]
    infer = synth.compose_infer_logprobs(logp, b.delta_noise, b.spikes)
    plants = harness.plant_band_tokens(b, logp, o["amin"], o["z_min"] - o["lse"], b.targets, infer)
    logp = np.where(b.targets == o["amin"], o["z_min"], o["z_y"]) - o["lse"]   # guard plants took argmin
    adv64 = oracle.group_advantages(b.rewards).reshape(-1)
    rep = oracle.icepop_loss(logp, infer.astype(np.float64), adv64, b.rollout_offsets, b.loss_mask, synth.ALPHA,
                             synth.BETA, synth.GUARD, b.loss_denominator, targets=b.targets, vocab=V)
    ref = _Ref(logp, o["entropy"], o["lse"], rep)
    c = harness.Case(b, None, None, infer, adv64.astype(np.float32), 1.0)
    c.plants = plants
    assert rep.guarded_rollouts >= 1 and len(plants) >= 12
    print(f"\n[{name}] T={T} kept {rep.kept_tokens} masked {rep.masked_low}+{rep.masked_high} "
          f"guarded {rep.guarded_rollouts} mean p_y {np.exp(logp).mean():.3f}")
    for dense in (False, True):
        g, dw = _gpu_step(c, dense)
        err = harness.compare(c, ref, g, check_grads=False)
        # gradients, given the gate (band flips take the GPU's coefficient, R13)
        coef = rep.coef.copy()
        flips = np.nonzero(g["keep"].astype(bool) != rep.keep)[0]
        coef[flips] = g["coef"][flips]
        dh_ref = coef[dh_rows, None] * (o["E"] - w64[b.targets[dh_rows]])
        err["d_hidden_row"] = harness.dh_row_error(g["dh"][dh_rows], dh_ref, coef[dh_rows], w64, b.targets[dh_rows])
        onehot = (b.targets[:, None] == dw_rows[None, :]).astype(np.float64)
        dw_ref = (coef[:, None] * (o["PS"] - onehot)).T @ h64
        dw_got = dw[torch.from_numpy(dw_rows).cuda()].cpu().numpy().astype(np.float64)
        err["d_w_vocab_tile"] = harness.dw_tile_error(dw_got, dw_ref, coef, h64, b.targets, row_ids=dw_rows)
        err["d_w_vocab_sample_fro"] = harness.rel_fro(dw_got, dw_ref)
        err["dw_colsum"] = g["dw_colsum"]
        zero = g["coef"] == 0
        err["dh_rows_zero_ok"] = bool(not g["dh"][zero].any())
        print(f"[{name}] {'dense' if dense else 'sparse'}: " + ", ".join(
            f"{k}={v:.3g}" if isinstance(v, float) else f"{k}={v}" for k, v in err.items()))
        assert err["d_hidden_row"] <= 1.0 and err["d_w_vocab_tile"] <= 1.0, err
        assert err["d_w_vocab_sample_fro"] <= harness.GRAD_RTOL, err
        assert err["dw_colsum"] < 1e-2 and err["dh_rows_zero_ok"], err
        del dw
        torch.cuda.empty_cache()


def test_hostio_full_size_bitwise_equals_device_path():
    """The e2e call bench.py times (rl_policy_loss_fwd_bwd_hostio: per-step inputs from
    pinned host memory, hidden rows uploaded in slabs under the forward, advantages by K0)
    at the glm16k size gives bit for bit what the device-resident call gives, so the
    full-size parity above covers the e2e path too."""
    wl = synth.CONFIGS["glm16k"]
    b = synth.make_batch(wl, 9)
    T, H, V = b.T, b.H, b.V
    R = wl.num_rollouts
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    w = bf(b.w_vocab)
    shape = rl.make_shape(T, H, V)
    # stored log-probs near the policy's own (this test compares two GPU paths, so the
    # recipe's reference log-prob may come from the GPU): ~1% masked, a few guarded rollouts
    lp0 = torch.empty(T, device=dev)
    rl.rl_logprob_fwd(shape, bf(b.hidden), w, torch.from_numpy(b.targets).to(dev), lp0)
    infer = synth.compose_infer_logprobs(lp0.cpu().numpy().astype(np.float64), b.delta_noise, b.spikes)
    params = rl.make_params(R, b.loss_denominator)
    outs = []
    for hostio in (False, True):
        report = rl.new_report(dev)
        dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        dw = torch.empty(V, H, device=dev)
        if hostio:
            pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
            rep = rl.rl_policy_loss_fwd_bwd_hostio(
                shape, params, wl.group_size, pin(b.hidden.view(np.int16)), w, pin(b.targets), pin(infer),
                pin(b.rewards.reshape(-1)), pin(b.rollout_offsets), pin(b.loss_mask), report=report, d_hidden=dh,
                d_w_vocab=dw).as_dict()
        else:
            adv = rl.rl_group_advantages(torch.from_numpy(b.rewards.reshape(-1).copy()).to(dev), wl.group_size)
            lp = torch.empty(T, device=dev)
            rl.rl_policy_loss_fwd_bwd(shape, params, bf(b.hidden), w, torch.from_numpy(b.targets).to(dev),
                                      torch.from_numpy(infer).to(dev), adv, torch.from_numpy(b.rollout_offsets).to(dev),
                                      torch.from_numpy(b.loss_mask).to(dev), report=report, logprob=lp, d_hidden=dh,
                                      d_w_vocab=dw)
            torch.cuda.synchronize()
            rep = rl.read_report(report).as_dict()
        outs.append((rep, dh.view(torch.int16).cpu(), dw.cpu()))
        del dw
        torch.cuda.empty_cache()
    assert outs[0][0] == outs[1][0]
    assert outs[0][0]["kept_tokens"] > T // 2 and outs[0][0]["masked_low"] > 0   # a real backward ran
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])
    print("\n[hostio glm16k] report", outs[1][0])


# ------------------------------------------- loss variants at full size (sampled rows)
VARIANTS_FULL = [
    dict(variant="cispo", alpha=0.8, beta=1.25, kl_tau=0.0, invt="scalar"),
    dict(variant="gspo", alpha=0.9, beta=1.1, kl_tau=0.0, invt="rows"),
    dict(variant="icepop", alpha=0.5, beta=5.0, kl_tau=0.375, kl_set="all", invt="rows"),
]


@pytest.mark.parametrize("cfg", VARIANTS_FULL, ids=lambda c: f"{c['variant']}-kl{c['kl_tau']}-{c['invt']}")
def test_full_size_variants_sampled_rows(cfg):
    """SURVEY §8 f2 at the glm16k size in the bench's launch configuration: CISPO (R16),
    GSPO (R17), the KL term (R19) and per-token temperature (R20) change only S3 (and the
    scale of z), so the GPU runs all 16384 rows and the loss sits on 512 sampled rows the
    oracle evaluates one by one: log-probs, gate, coef, loss, dH per row, dW per tile."""
    wl = synth.CONFIGS["glm16k"]
    b = synth.make_batch(wl, 21)
    T, H, V, R = b.T, b.H, b.V, wl.num_rollouts
    rng = np.random.default_rng(21)
    rows = np.sort(rng.choice(T, size=512, replace=False))
    invt_rows = rng.uniform(0.7, 1.5, T).astype(np.float32) if cfg["invt"] == "rows" else None
    invt_scalar = 1.0 / 0.7
    invt = invt_rows[rows].astype(np.float64) if invt_rows is not None else invt_scalar
    h64, w64 = oracle.bf16_to_f64(b.hidden[rows]), oracle.bf16_to_f64(b.w_vocab)
    Z = oracle.lm_logits(h64, w64, invt)
    _, _, lse0 = oracle.log_softmax_stats(Z, np.zeros(len(rows), np.int64))
    y = harness.sample_from_policy(Z, lse0, b.sample_u[rows])
    targets = b.targets.copy()
    targets[rows] = y
    logp0 = Z[np.arange(len(rows)), y] - lse0
    infer = np.full(T, -5.0, np.float32)
    infer[rows] = synth.compose_infer_logprobs(logp0, b.delta_noise[rows], np.zeros(len(rows), bool))
    lm = np.zeros(T, np.uint8)
    lm[rows] = 1
    rollout_of = np.repeat(np.arange(R), np.diff(b.rollout_offsets))
    sub_off = np.concatenate([[0], np.cumsum(np.bincount(rollout_of[rows], minlength=R))]).astype(np.int64)
    adv = oracle.group_advantages(b.rewards).reshape(-1)
    D = float(R) if cfg["variant"] == "gspo" else float(len(rows))
    kw = dict(alpha=cfg["alpha"], beta=cfg["beta"], guard_threshold=synth.GUARD, loss_denominator=D,
              inv_temperature=invt, backward=False, rollout_adv=adv, variant=cfg["variant"], kl_tau=cfg["kl_tau"],
              kl_set=cfg.get("kl_set", "masked"))
    ref = oracle.policy_loss_fwd_bwd(h64, w64, y, infer[rows].astype(np.float64), None, sub_off, None, **kw)
    # GPU: the whole batch through the C ABI (sparse backward, one 16384-row dU chunk)
    dev = "cuda"
    bf = lambda x: torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(dev)  # noqa: E731
    invt_dev = torch.from_numpy(invt_rows).to(dev) if invt_rows is not None else None
    shape = rl.make_shape(T, H, V, 0, V, invt_scalar if invt_rows is None else 1.0, inv_temperature_rows=invt_dev)
    params = rl.make_params(R, D, cfg["alpha"], cfg["beta"], synth.GUARD, cfg["variant"], kl_tau=cfg["kl_tau"],
                            kl_set=cfg.get("kl_set", "masked"))
    f32 = dict(dtype=torch.float32, device=dev)
    lp, ent, lse, coef = (torch.empty(T, **f32) for _ in range(4))
    keep = torch.empty(T, dtype=torch.uint8, device=dev)
    report = rl.new_report(dev)
    dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(V, H, **f32)
    rl.rl_policy_loss_fwd_bwd(shape, params, bf(b.hidden), bf(b.w_vocab), torch.from_numpy(targets).to(dev),
                              torch.from_numpy(infer).to(dev), torch.from_numpy(adv.astype(np.float32)).to(dev),
                              torch.from_numpy(b.rollout_offsets).to(dev), torch.from_numpy(lm).to(dev),
                              report=report, logprob=lp, entropy=ent, lse=lse, coef=coef, token_keep=keep,
                              d_hidden=dh, d_w_vocab=dw, dz_chunk_rows=T)
    torch.cuda.synchronize()
    rt = torch.from_numpy(rows).to(dev)
    g_lp, g_ent, g_coef = lp[rt].cpu().numpy(), ent[rt].cpu().numpy(), coef[rt].cpu().numpy()
    assert np.max(np.abs(g_lp - ref.logp)) <= harness.LOGP_TOL
    assert np.max(np.abs(g_ent - ref.entropy)) <= harness.LOGP_TOL
    rep = rl.read_report(report).as_dict()
    # the gate is exact outside the 1e-4 band (GSPO: of the rollout's sequence ratio)
    if cfg["variant"] == "gspo":
        v = ref.report.valid
        lr = np.where(v, ref.logp - infer[rows].astype(np.float64), 0.0)
        rsub = np.repeat(np.arange(R), np.diff(sub_off))
        n = np.bincount(rsub, weights=v.astype(float), minlength=R)
        s = np.exp(np.bincount(rsub, weights=lr, minlength=R) / np.maximum(n, 1))
        near = ((np.abs(s - cfg["alpha"]) <= harness.BAND) | (np.abs(s - cfg["beta"]) <= harness.BAND))[rsub]
    else:
        k = ref.report.ratio
        near = (np.abs(k - cfg["alpha"]) <= harness.BAND) | (np.abs(k - cfg["beta"]) <= harness.BAND) | (
            np.abs(k / synth.GUARD - 1.0) <= harness.BAND)
    differ = np.nonzero(np.abs(g_coef - ref.report.coef) > 1e-2 * np.abs(ref.report.coef) + 1e-9)[0]
    assert np.all(near[differ]), differ
    c_ref = ref.report.coef.copy()
    c_ref[differ] = g_coef[differ]
    slack = float(np.abs(g_coef[differ] - ref.report.coef[differ]).sum() * max(1.0, np.abs(ref.logp).max()))
    assert abs(rep["loss"] - ref.report.loss) <= harness.LOSS_TOL + slack, (rep["loss"], ref.report.loss)
    # gradients given the gate: dZ_t = invT_t coef_t (p_t - onehot)
    it = np.broadcast_to(np.asarray(invt, np.float64), (len(rows),))
    P = np.exp(Z - ref.lse[:, None])
    dh_ref = (it * c_ref)[:, None] * (P @ w64 - w64[y])
    err_h = harness.dh_row_error(dh[rt].float().cpu().numpy().astype(np.float64), dh_ref, c_ref, w64, y, it)
    blocks = np.arange(0, V, 256)
    ids = np.unique(np.concatenate([blocks + rng.integers(0, 256, len(blocks)), blocks + rng.integers(0, 256, len(blocks))]))
    ids = ids[ids < V]
    onehot = (y[:, None] == ids[None, :]).astype(np.float64)
    dw_ref = ((it * c_ref)[:, None] * (P[:, ids] - onehot)).T @ h64
    got = dw[torch.from_numpy(ids).to(dev)].cpu().numpy().astype(np.float64)
    err_w = harness.dw_tile_error(got, dw_ref, c_ref, h64, y, it, row_ids=ids)
    zero = ~np.isin(np.arange(T), rows)
    assert not dh.float()[torch.from_numpy(np.nonzero(zero)[0]).to(dev)].any().item()   # coef = 0 rows
    print(f"\n[{cfg['variant']} kl {cfg['kl_tau']} invT {cfg['invt']}] logp {np.max(np.abs(g_lp - ref.logp)):.3g} "
          f"coef differ {len(differ)} loss {rep['loss']:.6g} vs {ref.report.loss:.6g} dH row {err_h:.3g} dW tile {err_w:.3g}")
    assert err_h <= 1.0 and err_w <= 1.0
