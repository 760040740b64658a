"""Where the e2e (host-I/O) step loses time vs the device-resident step: wall-clock
per step of (a) the device call + sync, (b) the host-I/O call (H2D inside), (c) the
plain 134 MB pinned H2D alone."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402
import synth  # noqa: E402

wl = synth.CONFIGS["glm16k"]
dev = torch.device("cuda")
b = synth.make_batch_device(wl, 1, device=dev)
T, H, V, R = wl.tokens, wl.hidden, wl.vocab, wl.num_rollouts
shape = rl.make_shape(T, H, V)
infer = torch.clamp(-12.0 - b["delta"], max=0.0)
params = rl.make_params(R, float(T))
offsets = torch.from_numpy(b["offsets"]).to(dev)
lm = torch.from_numpy(b["loss_mask"]).to(dev)
adv = torch.zeros(R, device=dev)
rep = rl.new_report(dev)
lp = torch.empty(T, device=dev)
dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
dw = torch.empty(V, H, device=dev)
ws = rl.alloc_workspace(rl.rl_workspace_bytes_hostio(shape, R), dev)


def dev_step():
    rl.rl_policy_loss_fwd_bwd(shape, params, b["hidden"], b["w"], b["targets"], infer, adv, offsets, lm, report=rep,
                              logprob=lp, d_hidden=dh, d_w_vocab=dw, workspace=ws)
    torch.cuda.synchronize()


hp = b["hidden"].view(torch.int16).cpu().pin_memory()
tp, ip = b["targets"].cpu().pin_memory(), infer.cpu().pin_memory()
rp, op, mp_ = (torch.from_numpy(x).pin_memory() for x in (b["rewards"], b["offsets"], b["loss_mask"]))


def host_step():
    rl.rl_policy_loss_fwd_bwd_hostio(shape, params, wl.group_size, hp, b["w"], tp, ip, rp, op, mp_, report=rep,
                                     d_hidden=dh, d_w_vocab=dw, workspace=ws)


dst = torch.empty_like(b["hidden"])


def h2d():
    dst.view(torch.int16).copy_(hp, non_blocking=True)
    torch.cuda.synchronize()


for name, f in (("device step + sync", dev_step), ("hostio step", host_step), ("134 MB pinned H2D", h2d),
                ("device step + sync", dev_step), ("hostio step", host_step)):
    for _ in range(3):
        f()
    t = []
    for _ in range(10):
        t0 = time.perf_counter()
        f()
        t.append(time.perf_counter() - t0)
    print(f"{name:22s} median {np.median(t) * 1e3:7.2f} ms  min {min(t) * 1e3:7.2f} ms", flush=True)
