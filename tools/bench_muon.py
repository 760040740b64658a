"""Muon Newton-Schulz on the GLM-4.5-Air dW_vocab shape [151552, 4096]: librl (tcgen05)
vs the same 5-step quintic with torch.matmul (cuBLAS, bf16) on the same box.
FLOPs per step: 2 M N^2 (Gram) + 2 N^3 (Gram^2) + 2 M N^2 (X C)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402

M, N, STEPS = 151552, 4096, 5
g = torch.randn(M, N, device="cuda") * 1e-3
flops = STEPS * (4.0 * M * N * N + 2.0 * N ** 3)


def cublas_ns(G):
    a, b, c = 3.4445, -4.7750, 2.0315
    X = (G / (G.norm() + 1e-7)).bfloat16()
    for _ in range(STEPS):
        A = X.T @ X
        B = b * A + c * (A @ A)
        X = a * X + X @ B
    return X


def timeit(f, n=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
ws = rl.alloc_workspace(rl.load_library().rl_newton_schulz_workspace_bytes(M, N))
ms = timeit(lambda: rl.rl_newton_schulz(g, STEPS, out=out, workspace=ws))
ms_ref = timeit(lambda: cublas_ns(g))
ref = cublas_ns(g).float()
rel = float((out.float() - ref).norm() / ref.norm())
print(json.dumps({"shape": [M, N], "steps": STEPS, "librl_ms": ms, "librl_tflops": flops / ms / 1e9,
                  "cublas_torch_ms": ms_ref, "cublas_tflops": flops / ms_ref / 1e9,
                  "rel_diff_vs_cublas_path": rel}))

# per-launch breakdown of one call (CUDA events around each librl launch)
rl.rl_profile_enable(True)
rl.rl_profile_read()
rl.rl_newton_schulz(g, STEPS, out=out, workspace=ws)
torch.cuda.synchronize()
prof = rl.rl_profile_read()
rl.rl_profile_enable(False)
print(json.dumps([(k, round(m, 3)) for k, m in prof]))
