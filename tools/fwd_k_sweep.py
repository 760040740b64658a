"""Run the forward GEMM (K1) at H = 4096 and H = 8192 (same T x V) so one ncu pass
compares tensor-pipe activity at two tile lengths (per-tile-start cost check).
usage: python tools/fwd_k_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402

T, V = 16384, 151552
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
for H in (4096, 8192):
    h = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(V, H, generator=g, device=dev) * (4 / H ** 0.5)).to(torch.bfloat16)
    tg = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    shape = rl.make_shape(T, H, V)
    ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, 1), dev)
    lp = torch.empty(T, device=dev)
    for _ in range(2):
        rl.rl_logprob_fwd(shape, h, w, tg, lp, workspace=ws)
    torch.cuda.synchronize()
    del h, w, ws
print("ok")
