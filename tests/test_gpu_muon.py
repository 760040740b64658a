"""Newton-Schulz / Muon on the tcgen05 GEMMs vs the fp64 oracle (`-m gpu`).

Tolerance (R18): every iteration rounds X, A = X^T X and the polynomial
matrix C to bf16 (relative 2^-9 each) and the quintic amplifies perturbations of the
singular values by up to |p'| ~ 3.4, so after 5 steps the relative Frobenius error
stays below ~5e-2; singular values must also land in the quintic's band."""
import numpy as np
import pytest
import torch

from oracle import muon

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

NS_RTOL = 5e-2


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("M,N", [(3000, 512), (512, 3000), (1000, 200), (4096, 4096), (20000, 1024)])
def test_newton_schulz_vs_oracle(M, N):
    g = np.random.default_rng(M + N).standard_normal((M, N)).astype(np.float32)
    out = rl.rl_newton_schulz(torch.from_numpy(g).cuda(), 5)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().astype(np.float64)
    ref = muon.newton_schulz(g.astype(np.float64), 5)
    err = _rel(got, ref)
    print(M, N, err)
    assert err <= NS_RTOL
    sv = np.linalg.svd(got, compute_uv=False)
    assert sv.max() < 1.25   # the quintic overshoots to ~1.21 for tiny inputs (oracle pin)
    if max(M, N) >= 4 * min(M, N):   # well conditioned: every normalised singular value is >= 0.03
        assert sv.min() > 0.6


def test_muon_step_vs_oracle():
    rng = np.random.default_rng(11)
    M, N = 2048, 512
    th = rng.standard_normal((M, N)).astype(np.float32)
    g = rng.standard_normal((M, N)).astype(np.float32)
    m = (0.1 * rng.standard_normal((M, N))).astype(np.float32)
    t_th, t_g, t_m = (torch.from_numpy(x.copy()).cuda() for x in (th, g, m))
    rl.rl_muon_step(t_th, t_g, t_m, lr=0.02, mu=0.9, weight_decay=0.1)
    torch.cuda.synchronize()
    ref_th, ref_m = muon.muon_step(th, g, m, lr=0.02, mu=0.9, weight_decay=0.1)
    np.testing.assert_allclose(t_m.cpu().numpy(), ref_m, rtol=1e-6, atol=1e-6)
    upd_gpu = t_th.cpu().numpy().astype(np.float64) - th * (1 - 0.02 * 0.1)
    upd_ref = ref_th - th * (1 - 0.02 * 0.1)
    assert _rel(upd_gpu, upd_ref) <= NS_RTOL


def test_newton_schulz_rejects_bad_shapes():
    with pytest.raises(rl.RLError):
        rl.rl_newton_schulz(torch.zeros(10, 12, device="cuda"), 5)   # N % 8 != 0
    with pytest.raises(rl.RLError):
        rl.rl_newton_schulz(torch.zeros(16, 16, device="cuda"), 0)   # steps < 1
