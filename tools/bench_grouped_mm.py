"""PAPER.md Fig. 5 sweep on B200: grouped GEMM with hidden dim 4096 and MoE dim 1408,
tokens balanced over the experts, librl (tcgen05) vs torch._grouped_mm on the same box.
Prints one JSON line per (tokens, experts, projection)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402


def timeit(f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


HID, MOE = 4096, 1408
for tokens in (32768, 65536):
    for E in (8, 32, 128):
        for proj, (N, K) in (("up", (MOE, HID)), ("down", (HID, MOE))):
            a = torch.randn(tokens, K, device="cuda").to(torch.bfloat16)
            b = (torch.randn(E, N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
            off = torch.arange(0, E + 1, device="cuda", dtype=torch.int32) * (tokens // E)
            out = torch.empty(tokens, N, dtype=torch.bfloat16, device="cuda")
            flops = 2.0 * tokens * N * K
            ms = timeit(lambda: rl.rl_grouped_gemm(a, b, off, out=out))
            rec = {"tokens": tokens, "experts": E, "proj": proj, "N": N, "K": K, "librl_ms": ms,
                   "librl_tflops": flops / ms / 1e9}
            try:
                bt = b.transpose(-2, -1)
                ms_t = timeit(lambda: torch._grouped_mm(a, bt, offs=off[1:], out_dtype=torch.bfloat16))
                ref = torch._grouped_mm(a, bt, offs=off[1:], out_dtype=torch.bfloat16)
                rec.update(torch_grouped_mm_ms=ms_t, torch_tflops=flops / ms_t / 1e9,
                           rel_diff=float((out.float() - ref.float()).norm() / ref.float().norm()))
            except Exception as e:  # noqa: BLE001
                rec["torch_grouped_mm"] = f"unavailable: {type(e).__name__}: {e}"[:200]
            print(json.dumps(rec), flush=True)
