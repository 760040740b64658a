"""Multi-GPU compositions against the fp64 oracle of the WHOLE batch (`-m gpu`,
2-4 GPUs; skipped with fewer than 2).

The batch (sampled targets, guard spikes on argmin tokens, band-edge plants) is
built once in the parent from the oracle; every rank loads it, runs its share
through `parallel.py` on librl, and saves what it holds. The parent reassembles
the global outputs and holds them to `harness.compare`, i.e. to
`oracle.policy_loss_fwd_bwd` of the concatenated batch: logprob / entropy / lse,
keep (bit-exact outside the 1e-4 band), guard flags, counters, loss, dH per row
and dW per 256 x 512 tile. The gradient reduction is P:L92's (FSDP2 data
parallel) and P:L323's all-reduce, here NCCL or fused into the GEMM epilogue over
NVLS.

Data parallel: rank r holds prompt groups 2r, 2r+1 (whole groups: guard and
advantages stay local) with the global denominator D (R5); modes: NCCL, NVLS
all-reduce, NVLS reduce-scatter, NVLS with two micro-batches and three dU chunks
(accumulate, one deferred reduction), NVLS with an empty last rank (T = 0), NVLS
reduced by the epilogue warps (lag 2) instead of the communication warps.
Vocab parallel: W row-sharded; modes: NCCL, NVLS dense, NVLS sparse, NVLS sparse
with dU chunks.
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
G = 4
WL = synth.Workload("multi", 2 * WORLD, G, 96, 512, 3008, delta_sigma=0.5, spike_rate=3e-3)   # equal lengths
DP_MODES = ["nccl", "nvls", "nvls_rs", "nvls_micro", "nvls_empty", "nvls_lag2"]
VP_MODES = ["nccl", "nvls_dense", "nvls_sparse", "nvls_sparse_chunked"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    return harness.make_case(WL, 31, targets="sampled", plants=True)


def _save_case(path):
    c = _case()
    b = c.batch
    np.savez(path, hidden=b.hidden, w=b.w_vocab, targets=b.targets, infer=c.infer, rewards=b.rewards,
             offsets=b.rollout_offsets, loss_mask=b.loss_mask)
    return c


def _init(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    return dev


def _bf(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).to(dev)


def _report(eng):
    import paper_2512_16144_b200 as rl
    return rl.read_report(eng.report).as_dict()


def _dp_worker(rank, port, d):
    from paper_2512_16144_b200 import parallel
    dev = _init(rank, port)
    z = np.load(os.path.join(d, "case.npz"))
    off = z["offsets"]
    res = {}
    for mode in DP_MODES:
        # nvls_lag2: the epilogue warps reduce (rl_nvls_reduce.lag = 2, the round-1 schedule)
        # instead of the dedicated communication warps
        os.environ["RL_NVLS_LAG"] = "2" if mode == "nvls_lag2" else "0"
        micro = mode == "nvls_micro"
        empty = mode == "nvls_empty" and rank == WORLD - 1
        groups = [2 * rank, 2 * rank + 1]
        batches = [groups] if not micro else [[g] for g in groups]
        lm_mine = z["loss_mask"][off[groups[0] * G]:off[(groups[-1] + 1) * G]]
        if mode == "nvls_empty" and rank == WORLD - 1:
            lm_mine = lm_mine[:0]
        D = parallel.DataParallelPolicyLoss.global_denominator(torch.from_numpy(lm_mine.copy()).to(dev))
        out = {k: [] for k in ("logprob", "entropy", "lse", "coef", "keep", "guarded", "dh")}
        reps = []
        eng = None
        for j, gs in enumerate(batches):
            r0, r1 = gs[0] * G, (gs[-1] + 1) * G
            t0, t1 = int(off[r0]), int(off[r1])
            if empty:
                t1 = t0
            T = t1 - t0
            if eng is None:
                eng = parallel.DataParallelPolicyLoss(
                    parallel.LibrlPhases(), T=T, H=WL.hidden, V=WL.vocab, num_rollouts=r1 - r0, group_size=G,
                    loss_denominator=D, device=dev, nvls=mode != "nccl", reduce_scatter=mode == "nvls_rs",
                    dz_chunk_rows=128 if micro else 0)
            offs = np.zeros(r1 - r0 + 1, np.int32) if empty else (off[r0:r1 + 1] - t0).astype(np.int32)
            dw_buf = None if mode != "nccl" else torch.empty(WL.vocab, WL.hidden, device=dev)
            dw = eng.step(_bf(z["hidden"][t0:t1], dev), _bf(z["w"], dev),
                          torch.from_numpy(z["targets"][t0:t1].copy()).to(dev),
                          torch.from_numpy(z["infer"][t0:t1].copy()).to(dev),
                          torch.from_numpy(z["rewards"][gs].reshape(-1).copy()).to(dev),
                          torch.from_numpy(offs).to(dev),
                          torch.from_numpy(z["loss_mask"][t0:t1].copy()).to(dev), dw_buf,
                          accumulate=micro and j > 0, reduce=(not micro) or j == len(batches) - 1)
            torch.cuda.synchronize()
            for k, v in (("logprob", eng.logprob), ("entropy", eng.entropy), ("lse", eng.lse), ("coef", eng.coef),
                         ("keep", eng.keep), ("guarded", eng.guarded)):
                out[k].append(v.cpu().numpy().copy())
            out["dh"].append(eng.d_hidden.float().cpu().numpy().copy())
            reps.append(_report(eng))
        res[mode] = dict({k: np.concatenate(v) for k, v in out.items()}, dw=dw.cpu().numpy().copy(),
                         rep=np.array([sum(r[k] for r in reps) for k in sorted(reps[0])]),
                         rep_keys=np.array(sorted(reps[0])))
        dist.barrier()
    np.savez(os.path.join(d, f"dp{rank}.npz"), **{f"{m}__{k}": v for m, r in res.items() for k, v in r.items()})
    dist.barrier()
    dist.destroy_process_group()


def _vp_worker(rank, port, d):
    from paper_2512_16144_b200 import parallel
    dev = _init(rank, port)
    z = np.load(os.path.join(d, "case.npz"))
    T = len(z["targets"])
    res = {}
    for mode in VP_MODES:
        eng = parallel.VocabParallelPolicyLoss(
            parallel.LibrlPhases(dense_backward=mode == "nvls_dense"), T=T, H=WL.hidden, V_global=WL.vocab,
            num_rollouts=WL.num_rollouts, group_size=G, loss_denominator=float(z["loss_mask"].sum()), device=dev,
            nvls=mode != "nccl", dz_chunk_rows=512 if mode.endswith("chunked") else 0)
        lo, hi = eng.vocab_offset, eng.vocab_offset + eng.V_local
        dw = torch.empty(eng.V_local, WL.hidden, device=dev)
        dh = eng.step(_bf(z["hidden"], dev), _bf(z["w"][lo:hi], dev), torch.from_numpy(z["targets"]).to(dev),
                      torch.from_numpy(z["infer"]).to(dev), torch.from_numpy(z["rewards"].reshape(-1).copy()).to(dev),
                      torch.from_numpy(z["offsets"]).to(dev), torch.from_numpy(z["loss_mask"]).to(dev), dw)
        torch.cuda.synchronize()
        rep = _report(eng)
        res[mode] = dict(logprob=eng.logprob.cpu().numpy(), entropy=eng.entropy.cpu().numpy(),
                         lse=eng.lse.cpu().numpy(), coef=eng.coef.cpu().numpy(), keep=eng.keep.cpu().numpy(),
                         guarded=eng.guarded.cpu().numpy(), dh=dh.cpu().numpy().copy(), dw=dw.cpu().numpy(),
                         rep=np.array([rep[k] for k in sorted(rep)]), rep_keys=np.array(sorted(rep)))
        dist.barrier()
    np.savez(os.path.join(d, f"vp{rank}.npz"), **{f"{m}__{k}": v for m, r in res.items() for k, v in r.items()})
    dist.barrier()
    dist.destroy_process_group()


def _gpu_dict(r):
    rep = {str(k): float(v) if str(k) in ("loss", "mismatch_kl_sum") else int(v)
           for k, v in zip(r["rep_keys"], r["rep"])}
    return dict(logprob=r["logprob"], entropy=r["entropy"], lse=r["lse"], coef=r["coef"], keep=r["keep"],
                guarded=r["guarded"], report=rep, d_hidden=r["dh"].astype(np.float64),
                d_w_vocab=r["dw"].astype(np.float64))


def _load(path, mode):
    z = np.load(path)
    return {k.split("__", 1)[1]: z[k] for k in z.files if k.startswith(mode + "__")}


def _restrict(c, rows, rollouts):
    """The case on a subset of whole rollouts (the empty-rank batch)."""
    b = c.batch
    import dataclasses
    off = b.rollout_offsets[rollouts[0]:rollouts[-1] + 2] - b.rollout_offsets[rollouts[0]]
    nb = dataclasses.replace(b, hidden=b.hidden[rows], targets=b.targets[rows], loss_mask=b.loss_mask[rows],
                             rewards=b.rewards[rollouts[0] // G:(rollouts[-1] + 1) // G],
                             rollout_offsets=off.astype(np.int32), delta_noise=b.delta_noise[rows],
                             spikes=b.spikes[rows], sample_u=b.sample_u[rows])
    c2 = dataclasses.replace(c, batch=nb, h64=c.h64[rows], infer=c.infer[rows],
                             adv=c.adv[rollouts[0]:rollouts[-1] + 1])
    c2.plants = {r: v for r, v in c.plants.items() if r < len(rows)}
    return c2


@pytest.fixture(scope="module")
def dp_results(tmp_path_factory):
    d = tmp_path_factory.mktemp("dp")
    c = _save_case(str(d / "case.npz"))
    mp.start_processes(_dp_worker, args=(_port(), str(d)), nprocs=WORLD, start_method="spawn")
    return c, d


@pytest.fixture(scope="module")
def vp_results(tmp_path_factory):
    d = tmp_path_factory.mktemp("vp")
    c = _save_case(str(d / "case.npz"))
    mp.start_processes(_vp_worker, args=(_port(), str(d)), nprocs=WORLD, start_method="spawn")
    return c, d


@pytest.mark.parametrize("mode", DP_MODES)
def test_data_parallel_vs_oracle(dp_results, mode):
    c, d = dp_results
    ranks = [_load(str(d / f"dp{r}.npz"), mode) for r in range(WORLD)]
    if mode == "nvls_empty":
        # the last rank held no rows: the batch is the other ranks' rollouts
        R_used = 2 * G * (WORLD - 1)
        rows = np.arange(int(c.batch.rollout_offsets[R_used]))
        c = _restrict(c, rows, np.arange(R_used))
        assert len(ranks[-1]["logprob"]) == 0
    ref = harness.run_oracle(c)
    gpu = {k: np.concatenate([r[k] for r in ranks]) for k in ("logprob", "entropy", "lse", "coef", "keep")}
    gpu["guarded"] = np.concatenate([r["guarded"] for r in ranks])[:len(c.adv)]
    gpu["d_hidden"] = np.concatenate([r["dh"] for r in ranks]).astype(np.float64)
    if mode == "nvls_rs":
        import paper_2512_16144_b200 as rl
        S = rl.rl_nvls_shard_rows(WL.vocab, WORLD)
        gpu["d_w_vocab"] = np.concatenate([r["dw"] for r in ranks])[:WL.vocab].astype(np.float64)
        assert all(len(r["dw"]) == min(S, max(0, WL.vocab - i * S)) for i, r in enumerate(ranks))
    else:
        gpu["d_w_vocab"] = ranks[0]["dw"].astype(np.float64)
        for r in ranks[1:]:
            assert np.array_equal(r["dw"], ranks[0]["dw"])     # one reduced value on every rank
    keys = ranks[0]["rep_keys"]
    rep = {str(k): sum(float(r["rep"][i]) for r in ranks) for i, k in enumerate(keys)}
    gpu["report"] = {k: (v if k in ("loss", "mismatch_kl_sum") else int(round(v))) for k, v in rep.items()}
    err = harness.compare(c, ref, gpu)
    print("dp", mode, WORLD, err)


@pytest.mark.parametrize("mode", VP_MODES)
def test_vocab_parallel_vs_oracle(vp_results, mode):
    c, d = vp_results
    ranks = [_load(str(d / f"vp{r}.npz"), mode) for r in range(WORLD)]
    ref = harness.run_oracle(c)
    for r in ranks[1:]:   # S2/S3 run redundantly; dH is one reduced value on every rank
        for k in ("logprob", "entropy", "lse", "coef", "keep", "guarded", "dh"):
            assert np.array_equal(r[k], ranks[0][k]), k
    gpu = _gpu_dict(ranks[0])
    gpu["d_w_vocab"] = np.concatenate([r["dw"] for r in ranks]).astype(np.float64)
    err = harness.compare(c, ref, gpu)
    print("vp", mode, WORLD, err)
