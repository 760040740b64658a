"""MoE grouped GEMM on the tcgen05 kernels vs the fp64 oracle (`-m gpu`).
bf16 output: relative Frobenius error <= 4e-3 (one bf16 rounding, 2^-9, plus fp32
accumulation); rows of every group (incl. ragged / empty groups) and the N tail
(N = 1408 = 5.5 tiles) checked; guard bands prove no store leaves `out`."""
import numpy as np
import pytest
import torch

from oracle import moe

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402


def _bf(x):
    return torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("G,N,K,sizes", [
    (16, 1408, 4096, "balanced"),          # Fig. 5 up projection, 512 tokens per expert
    (8, 4096, 1408, "balanced"),           # down projection
    (12, 1408, 4096, "ragged"),            # uneven routing incl. empty experts
    (1, 256, 64, "one"),
])
def test_grouped_gemm_vs_oracle(G, N, K, sizes):
    rng = np.random.default_rng(G + N)
    if sizes == "balanced":
        n = np.full(G, 512)
    elif sizes == "ragged":
        n = rng.integers(0, 700, G)
        n[[2, 7]] = 0
        n[3] = 1
    else:
        n = np.array([300])
    off = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    rows = int(off[-1])
    a = _bf(rng.standard_normal((rows, K)))
    b = _bf(rng.standard_normal((G, N, K)) / np.sqrt(K))
    ref = moe.grouped_mm(a.float().numpy(), b.float().numpy(), off)
    guard = 4096
    buf = torch.full((rows * N + 2 * guard,), 7.0, dtype=torch.bfloat16, device="cuda")
    out = buf[guard:guard + rows * N].view(rows, N)
    rl.rl_grouped_gemm(a.cuda(), b.cuda(), torch.from_numpy(off).cuda(), out=out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().astype(np.float64)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(G, N, K, sizes, err)
    assert err <= 4e-3
    for g in range(G):   # every group individually (a wrong group mapping shows up here)
        r0, r1 = off[g], off[g + 1]
        if r1 > r0:
            assert np.linalg.norm(got[r0:r1] - ref[r0:r1]) <= 4e-3 * np.linalg.norm(ref[r0:r1]) + 1e-6
    assert bool((buf[:guard] == 7.0).all()) and bool((buf[-guard:] == 7.0).all())


def test_grouped_gemm_fused_rmsnorm():
    """RMSNorm fused into the expert GEMM: row scale 1/rms(x) on the fp32 accumulator,
    gamma folded into the weights; vs the oracle's normalise-then-multiply."""
    rng = np.random.default_rng(3)
    G, N, K = 8, 1408, 4096
    n = rng.integers(100, 600, G)
    off = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    rows = int(off[-1])
    x = _bf(rng.standard_normal((rows, K)) * rng.uniform(0.5, 3.0, (rows, 1)))
    gamma = rng.uniform(0.5, 1.5, K)
    w = rng.standard_normal((G, N, K)) / np.sqrt(K)
    ref = moe.grouped_mm_rmsnorm(x.float().numpy(), gamma, w, off, eps=1e-6)
    b = _bf(w * gamma[None, None, :])
    xs = x.cuda()
    scale = rl.rl_rms_inv(xs, 1e-6)
    out = rl.rl_grouped_gemm(xs, b.cuda(), torch.from_numpy(off).cuda(), row_scale=scale)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().astype(np.float64)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print("rmsnorm-fused", err)
    assert err <= 5e-3
