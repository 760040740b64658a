"""One process driving two GPUs (`-m gpu`, >= 2 GPUs): the same step on cuda:0 and then
on cuda:1 must both match the oracle and each other bit for bit. Kernel attributes
(the ~200 KB dynamic shared memory of the tcgen05 GEMMs) are per device; a library
that set them only for the first device it ran on fails its launches on the second.
The C ABI computes on the caller's current device and stream, so the caller selects
the device (`torch.cuda.device`)."""
import numpy as np
import pytest

import harness
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs 2 GPUs", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

WL = synth.Workload("two-dev", 2, 4, 150, 320, 2100, ragged=True, delta_sigma=0.6, spike_rate=5e-3)


def test_step_on_cuda1_after_cuda0_matches_oracle_and_is_identical():
    c = harness.make_case(WL, 41, targets="sampled", plants=True)
    ref = harness.run_oracle(c)
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            g = harness.run_gpu_step(c, device=f"cuda:{dev}")
        harness.compare(c, ref, g)
        outs.append(g)
    for k in ("logprob", "entropy", "lse", "coef", "keep", "guarded", "d_hidden", "d_w_vocab"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_newton_schulz_and_grouped_gemm_on_both_devices():
    gen = torch.Generator().manual_seed(3)
    g = torch.randn(1024, 512, generator=gen)
    a = torch.randn(700, 256, generator=gen).to(torch.bfloat16)
    b = torch.randn(3, 384, 256, generator=gen).to(torch.bfloat16)
    offs = torch.tensor([0, 300, 300, 700], dtype=torch.int32)
    res = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            d = f"cuda:{dev}"
            ns = rl.rl_newton_schulz(g.to(d), 5)
            gg = rl.rl_grouped_gemm(a.to(d), b.to(d), offs.to(d))
            torch.cuda.synchronize()
            res.append((ns.float().cpu(), gg.float().cpu()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
