"""Small end-to-end cases (tiny config, ragged tails, split phases) for compute-sanitizer.
usage: compute-sanitizer --tool memcheck python tests/sanitize_case.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import harness  # noqa: E402
import synth  # noqa: E402

for wl, kw in ((synth.CONFIGS["tiny"], {}),
               (synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8,
                               spike_rate=0.02), dict(tokens=333, vocab=1000, hidden=200))):
    c = harness.make_case(wl, 1, **kw)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c)
    print(wl.name, harness.compare(c, ref, gpu))
    gpu = harness.run_gpu_step(c, dh_f32=True, accumulate_dw=True, dw_init=None)
    gpu = harness.run_gpu_step(c, dense_backward=True, dz_chunk_rows=128)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16144_b200 as rl  # noqa: E402

# the f3 / f4 kernels: Newton-Schulz (split-K Gram), Muon, grouped GEMM with ragged groups, gamma fold
g = torch.randn(300, 136, device="cuda")
rl.rl_newton_schulz(g, 2)
th, m = torch.randn(300, 136, device="cuda"), torch.zeros(300, 136, device="cuda")
rl.rl_muon_step(th, g, m, lr=0.01)
a = torch.randn(333, 64, device="cuda").to(torch.bfloat16)
b = torch.randn(3, 96, 64, device="cuda").to(torch.bfloat16)
offs = torch.tensor([0, 100, 100, 333], dtype=torch.int32, device="cuda")
rl.rl_grouped_gemm(a, b, offs, row_scale=rl.rl_rms_inv(a))
rl.rl_fold_gamma(b, torch.rand(64, device="cuda"))
rl.rl_expert_load(offs, 333)
torch.cuda.synchronize()
print("sanitize cases ok")
