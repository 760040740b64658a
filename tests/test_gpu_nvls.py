"""The in-epilogue NVLink-multicast all-reduce (rl_nvls_reduce) against NCCL on
2-4 GPUs (`-m gpu`; skipped with fewer than 2 devices). DP: dW summed over ranks;
vocab-parallel: dH partials summed over ranks. Both must equal the NCCL
all-reduce of the same per-rank results up to fp32 summation order."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs 2 GPUs", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = min(4, torch.cuda.device_count())


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir, mode):
    import synth
    from paper_2512_16144_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    wl = synth.Workload("nv", 1, 4, 150, 512, 3008, ragged=True, delta_sigma=0.5)
    T = wl.tokens
    res = {}
    infer = None
    for nv in (False, False, True):
        if mode in ("dp", "dp_rs"):
            b = synth.make_batch_device(wl, 50 + rank, device=dev, tokens=T)
        else:
            Vl = wl.vocab // WORLD
            b = synth.make_batch_device(wl, 50, device=dev, tokens=T, vocab=Vl, vocab_offset=rank * Vl,
                                        vocab_total=wl.vocab)
        offs = torch.from_numpy(b["offsets"]).to(dev)
        lm = torch.from_numpy(b["loss_mask"]).to(dev)
        rw = torch.from_numpy(b["rewards"]).to(dev)
        inf = infer if infer is not None else torch.full((T,), -1.0, device=dev)
        if mode in ("dp", "dp_rs"):
            D = parallel.DataParallelPolicyLoss.global_denominator(lm)
            eng = parallel.DataParallelPolicyLoss(parallel.LibrlPhases(), T=T, H=wl.hidden, V=wl.vocab,
                                                  num_rollouts=wl.num_rollouts, group_size=wl.group_size,
                                                  loss_denominator=D, device=dev, nvls=nv,
                                                  reduce_scatter=nv and mode == "dp_rs")
            dw = torch.empty(wl.vocab, wl.hidden, device=dev)
            out = eng.step(b["hidden"], b["w"], b["targets"], inf, rw, offs, lm, None if nv else dw)
        else:
            eng = parallel.VocabParallelPolicyLoss(parallel.LibrlPhases(), T=T, H=wl.hidden, V_global=wl.vocab,
                                                   num_rollouts=wl.num_rollouts, group_size=wl.group_size,
                                                   loss_denominator=float(T), device=dev, nvls=nv)
            dw = torch.empty(eng.V_local, wl.hidden, device=dev)
            out = eng.step(b["hidden"], b["w"], b["targets"], inf, rw, offs, lm, dw)
        torch.cuda.synchronize()
        if infer is None:   # first pass: stored log-probs = own log-probs minus the drawn mismatch
            infer = torch.clamp(eng.logprob - b["delta"], max=0.0).contiguous()
            continue
        res["nvls" if nv else "nccl"] = out.cpu().numpy().copy()
    np.savez(os.path.join(out_dir, f"{mode}{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["dp", "vocab"])
def test_nvls_matches_nccl(tmp_path, mode):
    mp.start_processes(_worker, args=(_port(), str(tmp_path), mode), nprocs=WORLD, start_method="spawn")
    for r in range(WORLD):
        d = np.load(tmp_path / f"{mode}{r}.npz")
        a, b = d["nvls"], d["nccl"]
        assert np.abs(b).max() > 0
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    d = [np.load(tmp_path / f"{mode}{r}.npz")["nvls"] for r in range(WORLD)]
    assert all(np.array_equal(d[0], x) for x in d[1:])   # one reduced value, written to every replica


def test_nvls_reduce_scatter_matches_nccl_rows(tmp_path):
    """FSDP-consistent mode: rank r's returned shard equals rows [r S, (r+1) S) of the
    NCCL all-reduced dW (S = rl_nvls_shard_rows)."""
    import paper_2512_16144_b200 as rl
    mp.start_processes(_worker, args=(_port(), str(tmp_path), "dp_rs"), nprocs=WORLD, start_method="spawn")
    for r in range(WORLD):
        d = np.load(tmp_path / f"dp_rs{r}.npz")
        full, shard = d["nccl"], d["nvls"]
        S = rl.rl_nvls_shard_rows(full.shape[0], WORLD)
        ref = full[r * S:(r + 1) * S]
        assert shard.shape == ref.shape and np.abs(ref).max() > 0
        np.testing.assert_allclose(shard, ref, rtol=1e-5, atol=1e-6 * np.abs(full).max())


def _host_worker(rank, port, out_dir):
    import synth
    from paper_2512_16144_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    wl = synth.Workload("nv", 1, 4, 1500, 512, 3008, ragged=True, delta_sigma=0.5)   # T = 6000: three slabs
    T = wl.tokens
    Vl = wl.vocab // WORLD
    b = synth.make_batch_device(wl, 60, device=dev, tokens=T, vocab=Vl, vocab_offset=rank * Vl, vocab_total=wl.vocab)
    offs = torch.from_numpy(b["offsets"]).to(dev)
    lm = torch.from_numpy(b["loss_mask"]).to(dev)
    rw = torch.from_numpy(b["rewards"]).to(dev)
    inf = torch.full((T,), -1.0, device=dev)
    ok = []
    for nv in (False, True):
        eng = parallel.VocabParallelPolicyLoss(parallel.LibrlPhases(), T=T, H=wl.hidden, V_global=wl.vocab,
                                               num_rollouts=wl.num_rollouts, group_size=wl.group_size,
                                               loss_denominator=float(T), device=dev, nvls=nv)
        dw1 = torch.empty(eng.V_local, wl.hidden, device=dev)
        dw2 = torch.empty_like(dw1)
        a = eng.step(b["hidden"], b["w"], b["targets"], inf, rw, offs, lm, dw1).clone()
        lp1 = eng.logprob.clone()
        pin = lambda t: t.cpu().pin_memory()  # noqa: E731
        c = eng.step_host(pin(b["hidden"].view(torch.int16)), b["w"], pin(b["targets"]), pin(inf), pin(rw),
                          pin(offs), pin(lm), dw2).clone()
        torch.cuda.synchronize()
        ok.append(bool(torch.equal(a, c) and torch.equal(dw1, dw2) and torch.equal(lp1, eng.logprob)))
    np.save(os.path.join(out_dir, f"host{rank}.npy"), np.array(ok))
    dist.barrier()
    dist.destroy_process_group()


def test_vocab_parallel_step_host_equals_step(tmp_path):
    """step_host (pinned host inputs, hidden rows uploaded in slabs under the forward)
    gives step()'s outputs bit for bit, with NCCL and with the NVLS dH reduction."""
    mp.start_processes(_host_worker, args=(_port(), str(tmp_path)), nprocs=WORLD, start_method="spawn")
    for r in range(WORLD):
        assert np.load(tmp_path / f"host{r}.npy").all()
