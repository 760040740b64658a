"""Row-sharded Newton-Schulz (distributed Muon on d_w_vocab rows) on the
GPU (`-m gpu`): with one rank the three-phase sequence equals rl_newton_schulz bit for
bit; with two ranks each rank's rows match the fp64 oracle on the full matrix."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle.muon  # noqa: E402
import paper_2512_16144_b200 as rl  # noqa: E402
from paper_2512_16144_b200 import parallel  # noqa: E402

M, N = 3000, 512


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _G():
    return np.random.default_rng(8).standard_normal((M, N)).astype(np.float32)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_one_rank_equals_rl_newton_schulz_bitwise():
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        g = torch.from_numpy(_G()).cuda()
        a = parallel.newton_schulz_row_sharded(parallel.LibrlPhases(), g, steps=5)
        b = rl.rl_newton_schulz(g, 5)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", rank))
    rows = np.array_split(np.arange(M), 2)[rank]
    g = torch.from_numpy(_G()[rows].copy()).cuda()
    out = parallel.newton_schulz_row_sharded(parallel.LibrlPhases(), g, steps=5)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), out.float().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_ranks_match_oracle(tmp_path):
    mp.start_processes(_worker, args=(_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(2)])
    ref = oracle.muon.newton_schulz(_G().astype(np.float64), 5)
    assert _rel(got, ref) <= 5e-2                               # tests/test_gpu_muon.py's bf16 bound (R18)
    single = rl.rl_newton_schulz(torch.from_numpy(_G()).cuda(), 5).float().cpu().numpy()
    assert _rel(got, single) <= 2e-2                            # only the Gram's fp32 summation order differs
