"""Run each step GEMM once at the GLM-16k shape (after one warm-up step) so an
ncu --metrics pass can read its DRAM traffic. usage: python tools/gemm_traffic.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402

T, H, V = 16384, 4096, 151552
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
h = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16)
w = (torch.randn(V, H, generator=g, device=dev) * (4 / H ** 0.5)).to(torch.bfloat16)
tg = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
shape = rl.make_shape(T, H, V)
ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, 1), dev)
lp, lse = torch.empty(T, device=dev), torch.empty(T, device=dev)
coef = torch.full((T,), 1e-4, device=dev)
dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
dw = torch.empty(V, H, device=dev)
for _ in range(2):
    rl.rl_logprob_fwd(shape, h, w, tg, lp, None, lse, workspace=ws)
    rl.rl_bwd(shape, h, w, tg, lse, coef, d_hidden=dh, d_w_vocab=dw, workspace=ws)
torch.cuda.synchronize()
print("ok")
