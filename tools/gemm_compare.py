"""Sustained throughput of each step GEMM vs cuBLAS (torch.matmul) at the same
shape, on the same box, each looped for ~3 s so the clocks settle under the
power cap. Context for the roofline fraction: how close librl's tcgen05 kernels
are to the library GEMM when both pay the same power budget.

usage (GPU box): python tools/gemm_compare.py [--seconds 3]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_16144_b200 as rl  # noqa: E402


def clocks_during(fn, seconds):
    q = "clocks.sm,power.draw"
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0", "-lms", "200"],
                         stdout=subprocess.PIPE, text=True)
    lines = []
    t = threading.Thread(target=lambda: [lines.append(x) for x in p.stdout], daemon=True)
    t.start()
    n, ms = fn(seconds)
    p.terminate()
    t.join(timeout=2)
    vals = [tuple(float(v) for v in ln.split(",")) for ln in lines if ln.count(",") == 1]
    vals = vals[len(vals) // 4:]  # drop ramp-up
    sm = sorted(v[0] for v in vals)
    pw = sorted(v[1] for v in vals)
    return n, ms, (sm[len(sm) // 2] if sm else None), (pw[len(pw) // 2] if pw else None)


def loop(f, seconds):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    n = 0
    e0.record()
    while time.time() - t0 < seconds:
        f()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return n, e0.elapsed_time(e1) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--V", type=int, default=151552)
    a = ap.parse_args()
    T, H, V = a.T, a.H, a.V
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    h = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(V, H, generator=g, device=dev) * (4 / H ** 0.5)).to(torch.bfloat16)
    dz = (torch.randn(T, V, generator=g, device=dev) * 1e-4).to(torch.bfloat16)
    flops = 2.0 * T * V * H
    rows = []

    def rec(name, f):
        n, ms, sm, pw = clocks_during(lambda s: loop(f, s), a.seconds)
        rows.append({"gemm": name, "ms": ms, "tflops": flops / ms / 1e9, "sm_mhz": sm, "power_w": pw, "iters": n})
        print(json.dumps(rows[-1]), flush=True)

    # cuBLAS at the step's shapes
    rec("cublas Z = h W^T (K1/K4 shape)", lambda: torch.matmul(h, w.t()))
    rec("cublas dH = dU W (K5 shape)", lambda: torch.matmul(dz, w))
    rec("cublas dW = dU^T h (K6 shape)", lambda: torch.matmul(dz.t(), h))
    del dz
    # librl phases (K1+K2, then K4+K5+K6 together)
    shape = rl.make_shape(T, H, V)
    tg = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int64).to(torch.int32)
    lp, lse = torch.empty(T, device=dev), torch.empty(T, device=dev)
    ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, 1), dev)
    rec("librl K1+K2 (fwd, logits in TMEM)", lambda: rl.rl_logprob_fwd(shape, h, w, tg, lp, None, lse, workspace=ws))
    coef = torch.full((T,), 1e-4, device=dev)
    dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    dw = torch.empty(V, H, device=dev)
    # dU once, then each backward GEMM looped on its own (phase mask)
    rl.rl_bwd_ex(shape, h, w, tg, lse, coef, d_hidden=dh, d_w_vocab=dw, phases=rl.RL_BWD_DU, workspace=ws)
    for name, ph in (("librl K4 dU recompute", rl.RL_BWD_DU), ("librl K6 dW", rl.RL_BWD_DW),
                     ("librl K5 dH", rl.RL_BWD_DH)):
        rec(name, lambda ph=ph: rl.rl_bwd_ex(shape, h, w, tg, lse, coef, d_hidden=dh, d_w_vocab=dw, phases=ph,
                                             workspace=ws))
    rl.rl_profile_enable(True)
    rl.rl_profile_read()
    n, ms, sm, pw = clocks_during(lambda s: loop(lambda: rl.rl_bwd(shape, h, w, tg, lse, coef, d_hidden=dh,
                                                                      d_w_vocab=dw, workspace=ws), s), a.seconds)
    prof = rl.rl_profile_read(1 << 16)
    rl.rl_profile_enable(False)
    per = {}
    for k, m in prof:
        per.setdefault(k, []).append(m)
    for k, v in per.items():
        med = sorted(v)[len(v) // 2]
        rows.append({"gemm": f"librl {k} (in K4-K6 loop)", "ms": med, "tflops": flops / med / 1e9, "sm_mhz": sm,
                     "power_w": pw, "iters": len(v)})
        print(json.dumps(rows[-1]), flush=True)

if __name__ == "__main__":
    main()
