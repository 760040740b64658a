"""Run the fused step (rl_policy_loss_fwd_bwd, probability cache on by default) twice at the
GLM-16k shape on random data, for an ncu pass over its kernels: launches per step are K0, K1,
K2, K3, K3b, the compaction, K4 (from the cache), K6, K5 (a separate K1 computes the rollout
log-probs first, so every token is kept). usage: python tools/step_traffic.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402

T, H, V, R, G = 16384, 4096, 151552, 16, 16
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
h = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16)
w = (torch.randn(V, H, generator=g, device=dev) * (4 / H ** 0.5)).to(torch.bfloat16)
tg = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
shape = rl.make_shape(T, H, V)
params = rl.make_params(R, float(T))
infer = torch.empty(T, device=dev)
rewards = torch.rand(R, generator=g, device=dev)
offsets = torch.arange(0, T + 1, T // R, device=dev, dtype=torch.int32)
mask = torch.ones(T, dtype=torch.uint8, device=dev)
adv = rl.rl_group_advantages(rewards, G)
ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, R, 0), dev)
rl.rl_logprob_fwd(shape, h, w, tg, infer, workspace=ws)   # the rollout policy = this policy: every ratio 1, all kept
f32 = dict(dtype=torch.float32, device=dev)
lp, coef = torch.empty(T, **f32), torch.empty(T, **f32)
dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
dw = torch.empty(V, H, **f32)
rep = rl.new_report(dev)
for _ in range(2):
    rl.rl_policy_loss_fwd_bwd(shape, params, h, w, tg, infer, adv, offsets, mask, report=rep, logprob=lp, coef=coef,
                              d_hidden=dh, d_w_vocab=dw, workspace=ws)
torch.cuda.synchronize()
print("ok kept", int((coef != 0).sum().item()))
