"""Row-sharded Newton-Schulz at the GLM-4.5-Air dW shape [151552, 4096] over the ranks
of a torchrun job (5 steps; NCCL all-reduce of the 4096 x 4096 Gram per iteration).
Prints one JSON line from rank 0: ms per NS (CUDA events, max over ranks).
usage: torchrun --nproc-per-node N tools/bench_muon_dist.py"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402
from paper_2512_16144_b200 import parallel  # noqa: E402

M, N, STEPS = 151552, 4096, 5
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rows = M // world
g = torch.randn(rows, N, device=dev, generator=torch.Generator(device=dev).manual_seed(rank)) * 1e-3
ws = rl.alloc_workspace(rl.load_library().rl_newton_schulz_workspace_bytes(rows, N), dev)
out = torch.empty(rows, N, dtype=torch.bfloat16, device=dev)
ph = parallel.LibrlPhases()
for _ in range(2):
    parallel.newton_schulz_row_sharded(ph, g, STEPS, workspace=ws, out=out)
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
iters = 10
e0.record()
for _ in range(iters):
    parallel.newton_schulz_row_sharded(ph, g, STEPS, workspace=ws, out=out)
e1.record()
torch.cuda.synchronize()
t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
flops = STEPS * (4.0 * M * N * N + 2.0 * N ** 3)
if rank == 0:
    print(json.dumps({"shape": [M, N], "world": world, "rows_per_rank": rows, "steps": STEPS,
                      "ms": float(t.item()), "tflops_total": flops / (t.item() / 1e3) / 1e12,
                      "gram_allreduce_bytes_per_iter": N * N * 4}))
dist.destroy_process_group()
