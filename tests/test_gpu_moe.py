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
    # gamma folded into the expert weights on the device (once per optimizer step)
    b = rl.rl_fold_gamma(_bf(w).cuda(), torch.from_numpy(gamma.astype(np.float32)).cuda())
    xs = x.cuda()
    scale = rl.rl_rms_inv(xs, 1e-6)
    out = rl.rl_grouped_gemm(xs, b, torch.from_numpy(off).cuda(), row_scale=scale)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().astype(np.float64)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print("rmsnorm-fused", err)
    assert err <= 5e-3


def test_fold_gamma_vs_oracle_rounding():
    """out = bf16_rn(w * gamma): the fp32 product rounded once more to bf16 may differ
    from the exact product's rounding only on a double-rounding tie (<= 1 bf16 ulp)."""
    rng = np.random.default_rng(5)
    G, N, K = 3, 200, 1408
    w = _bf(rng.standard_normal((G, N, K)))
    gamma = rng.uniform(0.25, 2.0, K).astype(np.float32)
    got = rl.rl_fold_gamma(w.cuda(), torch.from_numpy(gamma).cuda())
    torch.cuda.synchronize()
    exact = w.double().numpy() * gamma.astype(np.float64)
    ref = torch.from_numpy(exact).to(torch.bfloat16).double().numpy()   # RN of the exact product
    g = got.double().cpu().numpy()
    diff = g != ref
    assert diff.mean() < 1e-3, diff.mean()
    assert np.all(np.abs(g - exact) <= np.abs(exact) * 2.0 ** -8 + 1e-30)
    inplace = w.cuda()
    rl.rl_fold_gamma(inplace, torch.from_numpy(gamma).cuda(), out=inplace)   # out may alias w
    assert torch.equal(inplace.cpu(), got.cpu())


@pytest.mark.parametrize("offs", [[0, 300, 300, 700], [0, 0, 0, 0], [0, 50, 40, 90, 90], [0, 7, 7, 7, 7, 7, 7, 8]])
def test_expert_load_vs_oracle(offs):
    """MaxViolation of the loads the grouped GEMM sees (offsets clamped,
    a decreasing pair counts as an empty group) vs oracle.moe.max_violation."""
    o = np.array(offs, np.int64)
    rows = int(o[-1])
    b = np.clip(o[:-1], 0, rows)
    e = np.maximum(np.clip(o[1:], 0, rows), b)
    load = (e - b).astype(np.float64)
    got = rl.rl_expert_load(torch.tensor(offs, dtype=torch.int32).cuda(), rows).cpu().numpy()
    assert got[0] == load.max() and got[1] == pytest.approx(load.mean(), rel=1e-7)
    want = moe.max_violation(load) if load.sum() > 0 else 0.0
    assert got[2] == pytest.approx(want, rel=1e-6, abs=1e-7)
