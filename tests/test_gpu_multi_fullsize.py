"""The fused NVLink-multicast collectives at BASELINE.json's full sizes, against the fp64
oracle (`-m gpu`, 2-4 GPUs; skipped with fewer than 2).

* Data parallel, the stress config's per-rank batch (16384 rows per rank, H = 4096,
  V = 151552, one G = 16 prompt group per rank): the whole 2.48 GB dW is all-reduced inside
  the dW GEMM's epilogue over NVLS, the GEMMs run over all rows (dense backward) as the
  bench times them.
* Vocab parallel, glm64k (65536 rows, W row-sharded): the dH partials are all-reduced
  inside the dH GEMM's epilogue over NVLS.

The oracle cannot afford every row of these batches, so `loss_mask` is 1 on a sample of
rows per rank (sampled targets, y ~ pi; stored log-probs with the
config's mismatch): every other row still runs through every GEMM with coef = 0, and the
outputs that depend on the sample are exact closed forms the oracle computes one by one —
logp / gate of the sampled rows, dH_t = coef_t (E_p[W] - W_{y_t}) per sampled row, and
dW[v] = sum over ALL ranks' sampled rows of coef_t (p_tv - [y_t = v]) h_t on sampled vocab
rows spread over every 256-row tile (per-tile error). The reduction is PAPER.md L92's
data-parallel gradient all-reduce (L323).
"""
import os
import socket

import numpy as np
import pytest
import torch

import harness
import oracle
import synth

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs 2 GPUs", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = min(4, torch.cuda.device_count())
DP_WL = synth.Workload("stress-rank", 1, 16, 1024, 4096, 151552, delta_sigma=1.0, spike_rate=1e-4)
VP_WL = synth.CONFIGS["glm64k"]
W_SEED = 7
N_SAMPLE = 256


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bf(bits, dev):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def _plan(b, w64, seed, n=N_SAMPLE):
    """Sampled rows with targets drawn from the policy and their stored log-probs."""
    rows = np.sort(np.random.default_rng(seed).choice(b.T, size=n, replace=False))
    h64 = oracle.bf16_to_f64(b.hidden[rows])
    Z = oracle.lm_logits(h64, w64)
    _, _, lse = oracle.log_softmax_stats(Z, np.zeros(n, np.int64))
    y = harness.sample_from_policy(Z, lse, b.sample_u[rows])
    amin = np.argmin(Z, axis=1)
    y = np.where(b.spikes[rows], amin, y).astype(np.int32)
    logp = Z[np.arange(n), y] - lse
    targets = b.targets.copy()
    targets[rows] = y
    infer = np.full(b.T, -5.0, np.float32)
    infer[rows] = synth.compose_infer_logprobs(logp, b.delta_noise[rows], b.spikes[rows])
    lm = np.zeros(b.T, np.uint8)
    lm[rows] = 1
    return dict(rows=rows, targets=targets, infer=infer, loss_mask=lm, h64=h64, Z=Z, lse=lse, y=y)


def _sampled_gate(b, plan, adv, D):
    """Eq.1 / Eq.2 / guard of the sampled rows: the rollout structure re-based to them
    (the other rows have loss_mask 0: no loss, no guard participation, reading R4/R5)."""
    rows = plan["rows"]
    rollout_of = np.repeat(np.arange(len(b.rollout_offsets) - 1), np.diff(b.rollout_offsets))
    counts = np.bincount(rollout_of[rows], minlength=len(b.rollout_offsets) - 1)
    sub_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    logp = plan["Z"][np.arange(len(rows)), plan["y"]] - plan["lse"]
    rep = oracle.icepop_loss(logp, plan["infer"][rows].astype(np.float64), adv, sub_off, None, synth.ALPHA,
                             synth.BETA, synth.GUARD, D)
    return logp, rep


def _band(rep):
    k, v = rep.ratio, rep.valid
    return v & ((np.abs(k - synth.ALPHA) <= harness.BAND) | (np.abs(k - synth.BETA) <= harness.BAND)
                | (np.abs(k / synth.GUARD - 1.0) <= harness.BAND))


def _dw_rows(V, seed):
    rng = np.random.default_rng(seed)
    blocks = np.arange(0, V, 256)
    r = np.unique(np.concatenate([blocks + rng.integers(0, 256, size=len(blocks)),
                                  blocks + rng.integers(0, 256, size=len(blocks))]))
    return r[r < V]


# --------------------------------------------------------------------------- DP
def _dp_worker(rank, port, d):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    from paper_2512_16144_b200 import parallel
    b = synth.make_batch(DP_WL, 300 + rank, w_seed=W_SEED)
    z = np.load(os.path.join(d, f"plan{rank}.npz"))
    D = float(z["D"])
    eng = parallel.DataParallelPolicyLoss(parallel.LibrlPhases(dense_backward=True), T=b.T, H=b.H, V=b.V,
                                          num_rollouts=DP_WL.num_rollouts, group_size=DP_WL.group_size,
                                          loss_denominator=D, device=dev, nvls=True)
    dw = eng.step(_bf(b.hidden, dev), _bf(b.w_vocab, dev), torch.from_numpy(z["targets"]).to(dev),
                  torch.from_numpy(z["infer"]).to(dev), torch.from_numpy(b.rewards.reshape(-1).copy()).to(dev),
                  torch.from_numpy(b.rollout_offsets).to(dev), torch.from_numpy(z["loss_mask"]).to(dev))
    torch.cuda.synchronize()
    rows = torch.from_numpy(z["rows"]).to(dev)
    dwr = torch.from_numpy(z["dw_rows"]).to(dev)
    import paper_2512_16144_b200 as rl
    rep = rl.read_report(eng.report).as_dict()
    np.savez(os.path.join(d, f"out{rank}.npz"), logprob=eng.logprob[rows].cpu().numpy(),
             coef=eng.coef[rows].cpu().numpy(), keep=eng.keep[rows].cpu().numpy(),
             dh=eng.d_hidden[rows].float().cpu().numpy(), dw=dw[dwr].cpu().numpy(),
             dh_rest_zero=np.array(bool((eng.d_hidden.float().abs().sum(1) != 0).sum().item() <= len(z["rows"]))),
             loss=np.array(rep["loss"]))
    dist.barrier()
    dist.destroy_process_group()


def test_dp_nvls_full_size_vs_oracle(tmp_path):
    d = str(tmp_path)
    w_batch = synth.make_batch(DP_WL, 300, w_seed=W_SEED)
    w64 = oracle.bf16_to_f64(w_batch.w_vocab)
    dw_rows = _dw_rows(DP_WL.vocab, 5)
    plans, batches = [], []
    for r in range(WORLD):
        b = w_batch if r == 0 else synth.make_batch(DP_WL, 300 + r, with_weights=False)
        plan = _plan(b, w64, 40 + r)
        plans.append(plan)
        batches.append(b)
    D = float(N_SAMPLE * WORLD)   # the global loss-token count of the step (R5)
    for r, (b, plan) in enumerate(zip(batches, plans)):
        np.savez(os.path.join(d, f"plan{r}.npz"), rows=plan["rows"], targets=plan["targets"], infer=plan["infer"],
                 loss_mask=plan["loss_mask"], D=D, dw_rows=dw_rows)
    mp.start_processes(_dp_worker, args=(_port(), d), nprocs=WORLD, start_method="spawn")
    outs = [np.load(os.path.join(d, f"out{r}.npz")) for r in range(WORLD)]
    dw_ref = np.zeros((len(dw_rows), w64.shape[1]))
    coef_all, h_all, y_all = [], [], []
    loss_ref = 0.0
    for r, (b, plan, o) in enumerate(zip(batches, plans, outs)):
        adv = oracle.group_advantages(b.rewards).reshape(-1)
        logp, rep = _sampled_gate(b, plan, adv, D)
        loss_ref += rep.loss
        assert np.max(np.abs(o["logprob"] - logp)) <= harness.LOGP_TOL
        band = _band(rep)
        flips = np.nonzero(o["keep"].astype(bool) != rep.keep)[0]
        assert np.all(band[flips]), flips
        coef = rep.coef.copy()
        coef[flips] = o["coef"][flips]          # the gradient is unique given the gate (R13)
        P = np.exp(plan["Z"] - plan["lse"][:, None])
        dh_ref = coef[:, None] * (P @ w64 - w64[plan["y"]])
        err = harness.dh_row_error(o["dh"].astype(np.float64), dh_ref, coef, w64, plan["y"])
        assert err <= 1.0, (r, err)
        assert bool(o["dh_rest_zero"])
        onehot = (plan["y"][:, None] == dw_rows[None, :]).astype(np.float64)
        dw_ref += (coef[:, None] * (P[:, dw_rows] - onehot)).T @ plan["h64"]
        coef_all.append(coef), h_all.append(plan["h64"]), y_all.append(plan["y"])
    loss_gpu = sum(float(o["loss"]) for o in outs)
    assert abs(loss_gpu - loss_ref) <= harness.LOSS_TOL
    for o in outs[1:]:
        assert np.array_equal(o["dw"], outs[0]["dw"])       # one reduced value on every rank
    tile = harness.dw_tile_error(outs[0]["dw"].astype(np.float64), dw_ref, np.concatenate(coef_all),
                                 np.concatenate(h_all), np.concatenate(y_all), row_ids=dw_rows)
    fro = harness.rel_fro(outs[0]["dw"], dw_ref)
    print(f"\n[dp nvls x{WORLD}] loss {loss_gpu:.6g} vs {loss_ref:.6g}, d_w_vocab_tile {tile:.3g}, fro {fro:.3g}")
    assert tile <= 1.0 and fro <= harness.GRAD_RTOL


# --------------------------------------------------------------------------- VP
def _vp_worker(rank, port, d):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    from paper_2512_16144_b200 import parallel
    b = synth.make_batch(VP_WL, 400, w_seed=W_SEED)
    z = np.load(os.path.join(d, "plan.npz"))
    eng = parallel.VocabParallelPolicyLoss(parallel.LibrlPhases(dense_backward=True), T=b.T, H=b.H, V_global=b.V,
                                           num_rollouts=VP_WL.num_rollouts, group_size=VP_WL.group_size,
                                           loss_denominator=float(z["D"]), device=dev, nvls=True,
                                           dz_chunk_rows=16384)
    lo, hi = eng.vocab_offset, eng.vocab_offset + eng.V_local
    dw = torch.empty(eng.V_local, b.H, device=dev)
    dh = eng.step(_bf(b.hidden, dev), _bf(b.w_vocab[lo:hi], dev), torch.from_numpy(z["targets"]).to(dev),
                  torch.from_numpy(z["infer"]).to(dev), torch.from_numpy(b.rewards.reshape(-1).copy()).to(dev),
                  torch.from_numpy(b.rollout_offsets).to(dev), torch.from_numpy(z["loss_mask"]).to(dev), dw)
    torch.cuda.synchronize()
    rows = torch.from_numpy(z["rows"]).to(dev)
    mine = z["dw_rows"][(z["dw_rows"] >= lo) & (z["dw_rows"] < hi)]
    np.savez(os.path.join(d, f"out{rank}.npz"), logprob=eng.logprob[rows].cpu().numpy(),
             coef=eng.coef[rows].cpu().numpy(), keep=eng.keep[rows].cpu().numpy(),
             dh=dh[rows].float().cpu().numpy(), dw=dw[torch.from_numpy(mine - lo).to(dev)].cpu().numpy(), dw_ids=mine)
    dist.barrier()
    dist.destroy_process_group()


def test_vocab_parallel_nvls_full_size_vs_oracle(tmp_path):
    d = str(tmp_path)
    b = synth.make_batch(VP_WL, 400, w_seed=W_SEED)
    w64 = oracle.bf16_to_f64(b.w_vocab)
    plan = _plan(b, w64, 77, n=2 * N_SAMPLE)
    dw_rows = _dw_rows(VP_WL.vocab, 6)
    D = float(len(plan["rows"]))
    np.savez(os.path.join(d, "plan.npz"), rows=plan["rows"], targets=plan["targets"], infer=plan["infer"],
             loss_mask=plan["loss_mask"], D=D, dw_rows=dw_rows)
    mp.start_processes(_vp_worker, args=(_port(), d), nprocs=WORLD, start_method="spawn")
    outs = [np.load(os.path.join(d, f"out{r}.npz")) for r in range(WORLD)]
    adv = oracle.group_advantages(b.rewards).reshape(-1)
    logp, rep = _sampled_gate(b, plan, adv, D)
    o = outs[0]
    for x in outs[1:]:   # S2/S3 run redundantly; dH is one reduced value on every rank
        for k in ("logprob", "coef", "keep", "dh"):
            assert np.array_equal(x[k], o[k]), k
    assert np.max(np.abs(o["logprob"] - logp)) <= harness.LOGP_TOL
    flips = np.nonzero(o["keep"].astype(bool) != rep.keep)[0]
    assert np.all(_band(rep)[flips]), flips
    coef = rep.coef.copy()
    coef[flips] = o["coef"][flips]
    P = np.exp(plan["Z"] - plan["lse"][:, None])
    dh_ref = coef[:, None] * (P @ w64 - w64[plan["y"]])
    err = harness.dh_row_error(o["dh"].astype(np.float64), dh_ref, coef, w64, plan["y"])
    ids = np.concatenate([x["dw_ids"] for x in outs])
    got = np.concatenate([x["dw"] for x in outs]).astype(np.float64)
    onehot = (plan["y"][:, None] == ids[None, :]).astype(np.float64)
    dw_ref = (coef[:, None] * (P[:, ids] - onehot)).T @ plan["h64"]
    tile = harness.dw_tile_error(got, dw_ref, coef, plan["h64"], plan["y"], row_ids=ids)
    print(f"\n[vp nvls x{WORLD}] T={b.T} d_hidden_row {err:.3g} d_w_vocab_tile {tile:.3g}")
    assert err <= 1.0 and tile <= 1.0
