"""NCCL collective timing for the dW / dH exchange sizes (run under torchrun)."""
import os

import torch
import torch.distributed as dist

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
for name, numel, dt in (("dW fp32", 151552 * 4096, torch.float32), ("dW bf16", 151552 * 4096, torch.bfloat16),
                        ("dH fp32 64k", 65536 * 4096, torch.float32)):
    x = torch.ones(numel, dtype=dt, device="cuda")
    for op in ("all_reduce", "reduce_scatter"):
        out = torch.empty(numel // world, dtype=dt, device="cuda")
        f = (lambda: dist.all_reduce(x)) if op == "all_reduce" else (lambda: dist.reduce_scatter_tensor(out, x))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        nbytes = numel * x.element_size()
        bus = nbytes * (2 if op == "all_reduce" else 1) * (world - 1) / world / (ms / 1e3) / 1e9
        if rank == 0:
            print(f"{name:12s} {op:15s} {nbytes/1e9:.2f} GB  {ms:7.2f} ms  busbw {bus:6.0f} GB/s", flush=True)
dist.destroy_process_group()
