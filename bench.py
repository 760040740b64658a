#!/usr/bin/env python
"""bench.py — policy-loss fwd+bwd tokens/s on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over one
packed micro-batch per rank: group advantages, LM-head GEMM with the online
log-softmax epilogue, partial merge, Eq.1/Eq.2/guard coefficients, and the
backward (dU recompute, dH = dU W, dW = dU^T h), plus the step's collectives.

  N = 1 : GLM-4.5-Air-shaped 16k-token micro-batch (H 4096, V 151552), 1 GPU.
  N > 1 : default: the same GLM-16k micro-batch on every rank (data parallel, weak
          scaling; rank r draws seed 1000 + r), dW all-reduce every step (fused in
          the dW GEMM epilogue over NVLS when multicast is available, else NCCL).
          --config stress: 16k tokens / rank, one G=16 group per rank, heavy
          off-policy log-probs (about a quarter of the tokens masked by Eq.2).
          --config glm64k: vocab-parallel (strong scaling) 64k tokens, W sharded,
          partials all-gather + dH all-reduce (NCCL).

`--impl reference` times the fp64 CPU oracle (the tier's reference arm) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "policy-loss fwd+bwd tokens/s at 1/2/4/8 B200; % of GEMM/HBM roofline"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", ",".join(str(g) for g in self.gpus), "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------- utils
def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def emit(d):
    print(json.dumps(d), flush=True)


def workload_for(args, world):
    import synth
    if args.config != "auto":
        name = args.config
    else:
        name = "glm16k"
    wl = synth.CONFIGS[name]
    return name, wl


# ---------------------------------------------------- reference (oracle) arm
def oracle_sample(wl, sample_tokens, seed=0):
    """A bounded slice of the workload for the fp64 oracle: `sample_tokens` packed
    rows (whole rollouts of the config's length, at least one), the full H and V."""
    import oracle
    import synth
    R = max(1, sample_tokens // wl.rollout_len) if sample_tokens >= wl.rollout_len else 1
    sub = synth.Workload(wl.name + "-sample", 1, max(2, R), max(1, sample_tokens // max(2, R)), wl.hidden,
                         wl.vocab, sigma_z=wl.sigma_z, delta_sigma=wl.delta_sigma, spike_rate=wl.spike_rate)
    b = synth.make_batch(sub, seed)
    h64, w64 = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    infer = synth.compose_infer_logprobs(np.full(b.T, -5.0), b.delta_noise, b.spikes).astype(np.float64)
    return b, h64, w64, infer


def run_oracle_step(b, h64, w64, infer):
    import oracle
    return oracle.policy_loss_fwd_bwd(h64, w64, b.targets, infer, b.rewards, b.rollout_offsets, b.loss_mask)


def host_info():
    """CPU model and BLAS library/threads of the host that times the oracle."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        from threadpoolctl import threadpool_info
        libs = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if libs:
            blas = f"{libs[0].get('internal_api')} {libs[0].get('version')} ({libs[0].get('num_threads')} threads)"
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "blas": blas}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 0) for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(max(n)) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def cpu_baseline(wl, budget_s=15.0):
    """Time the oracle as it stands on a bounded sample; returns the cpu_baseline object.
    Two calibration calls (the first pays BLAS warm-up) size the sample so the timed
    call takes about `budget_s`; the per-call fixed cost (the fp64 dW [V, H]) is kept."""
    def timed(tok):
        b, h64, w64, infer = oracle_sample(wl, tok)
        t0 = time.perf_counter()
        run_oracle_step(b, h64, w64, infer)
        return b, time.perf_counter() - t0

    timed(64)
    _, t64 = timed(64)
    _, t256 = timed(256)
    per_tok = max((t256 - t64) / 192, 1e-6)
    fixed = max(t64 - 64 * per_tok, 0.0)
    tok = int(min(8192, max(64, (budget_s - fixed) / per_tok)))
    tok = 1 << int(math.log2(tok))
    b, dt = timed(tok)
    return {"value": b.T / dt, "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
            "sample": f"{b.T} tokens ({len(b.rollout_offsets) - 1} rollouts) of the {wl.name} shape "
                      f"(H={wl.hidden}, V={wl.vocab}), full fwd+bwd in fp64 numpy; bf16->fp64 decode excluded; "
                      f"{dt:.1f} s", **host_info()}


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    name, wl = workload_for(args, world)
    try:  # torchrun pins OMP/BLAS to 1 thread; the oracle is timed on all host cores
        from threadpoolctl import threadpool_limits
        threadpool_limits(os.cpu_count())
    except Exception:  # noqa: BLE001
        pass
    # tokens per reference step: 256, or 64 when many steps are asked for (each step also
    # pays a fixed ~1-2 s for the fp64 [V, H] dW), so K + W steps end within minutes
    ref_tokens = args.ref_tokens or (256 if args.steps + args.warmup <= 43 else 64)
    b, h64, w64, infer = oracle_sample(wl, ref_tokens)
    for _ in range(args.warmup):
        run_oracle_step(b, h64, w64, infer)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run_oracle_step(b, h64, w64, infer)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    v = b.T / dt
    cb = {"value": v, "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
          "sample": f"{b.T} tokens per step of the {wl.name} shape (H={wl.hidden}, V={wl.vocab}), fp64 numpy oracle",
          **host_info()}
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
          "config": {"workload": name, "T_sample": b.T, "H": wl.hidden, "V": wl.vocab},
          "cpu_baseline": cb, "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}})
    return 0


# ------------------------------------------------------------------ our arm
def _setup(args):
    """Process group, collective, per-rank workload and its synthetic batch."""
    import types

    import torch
    import torch.distributed as dist

    import paper_2512_16144_b200 as rl
    import synth

    r = types.SimpleNamespace()
    r.rank, r.world, r.local = env_rank()
    if r.world != args.gpus:
        args.gpus = r.world
    torch.cuda.set_device(r.local)
    r.dev = dev = torch.device("cuda", r.local)
    if r.world > 1:
        dist.init_process_group("nccl", device_id=dev)
    r.name, r.wl = workload_for(args, r.world)
    if args.tokens:
        # A/B knob: the same shape with another micro-batch size (rollouts keep their count)
        import dataclasses
        r.wl = dataclasses.replace(r.wl, rollout_len=max(1, int(args.tokens) // r.wl.num_rollouts))
    if args.delta_sigma is not None:
        # A/B knob: the trainer-inference mismatch of the stress config on another shape
        # (e.g. vocab-parallel glm64k with ~43% of rows masked, for the sparse backward)
        import dataclasses
        r.wl = dataclasses.replace(r.wl, delta_sigma=float(args.delta_sigma))
    if args.collective == "auto":
        args.collective = "nccl"
        if r.world > 1:
            import torch.distributed._symmetric_memory as symm_mem
            try:
                probe = symm_mem.empty(1024, dtype=torch.float32, device=dev)
                ok = torch.tensor([1 if symm_mem.rendezvous(probe, dist.group.WORLD.group_name).multicast_ptr
                                   else 0], device=dev)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                args.collective = "nvls" if ok.item() else "nccl"
            except Exception:  # noqa: BLE001 - no symmetric memory / multicast here: NCCL
                args.collective = "nccl"
    r.vocab_par = r.name == "glm64k" and r.world > 1
    r.mode = "vocab" if r.vocab_par else "dp"
    r.H, r.Vt = r.wl.hidden, r.wl.vocab
    if r.name == "stress":
        # 16k tokens and one G=16 prompt group per rank (the guard and advantages stay local)
        r.T = r.wl.tokens // r.wl.n_ranks
        r.wl_rank = synth.Workload("stress-rank", 1, r.wl.group_size, r.wl.rollout_len, r.H, r.Vt,
                                   delta_sigma=r.wl.delta_sigma, spike_rate=r.wl.spike_rate)
    else:
        r.T = r.wl.tokens
        r.wl_rank = r.wl
    if r.vocab_par:
        assert r.Vt % r.world == 0
        r.V_local, r.v_off = r.Vt // r.world, r.rank * (r.Vt // r.world)
    else:
        r.V_local, r.v_off = r.Vt, 0
    seed = 1000 + (0 if r.vocab_par else r.rank)
    r.b = b = synth.make_batch_device(r.wl_rank, seed, device=dev, tokens=r.T, vocab=r.V_local,
                                      vocab_offset=r.v_off, vocab_total=r.Vt)
    r.R = len(b["offsets"]) - 1
    r.shape = rl.make_shape(r.T, r.H, r.V_local, r.v_off, r.Vt)
    r.targets = b["targets"]
    r.offsets = torch.from_numpy(b["offsets"]).to(dev)
    r.loss_mask = torch.from_numpy(b["loss_mask"]).to(dev)
    r.rewards = torch.from_numpy(b["rewards"]).to(dev)
    D = float(b["loss_mask"].sum())
    if r.world > 1 and not r.vocab_par:
        t = torch.tensor([D], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        D = float(t.item())
    r.D = D
    r.params = rl.make_params(r.R, D)
    # dU in 16k-row chunks: keeps K5/K6's per-wave working set inside L2 (the K = T
    # reduction of K6 at 64k rows loses ~20% to HBM re-reads otherwise)
    r.chunk = 0 if r.T <= 16384 else 16384
    if args.dz_chunk >= 0:
        r.chunk = args.dz_chunk
    return r


def _sample_targets(r, seed=77, chunk=1024):
    """Rollout targets sampled from the policy itself (y ~ pi; SURVEY
    §8(d)): Gumbel-max over the logits h W^T of each row, computed here with torch as
    the inference engine's stand-in (input generation, outside the timed region; the
    measured path never sees how the targets were made). Guard-spike rows get the row's
    least likely token instead, so the guard trips although sampled targets are probable.
    Vocab-parallel ranks take the max / min over their shard and agree on the global one
    with one all-gather."""
    import torch
    import torch.distributed as dist

    g = torch.Generator(device=r.dev)
    g.manual_seed(seed * 1009 + r.rank)
    h, w = r.b["hidden"], r.b["w"]
    best = torch.empty(r.T, 4, dtype=torch.float32, device=r.dev)   # (max z+gumbel, its id, min z, its id)
    for c0 in range(0, r.T, chunk):
        c1 = min(r.T, c0 + chunk)
        z = torch.matmul(h[c0:c1], w.t()).float()
        u = torch.rand(z.shape, generator=g, device=r.dev).clamp_(1e-20, 1.0)
        zg = z - torch.log(-torch.log(u))
        mx, ix = zg.max(dim=1)
        mn, jn = z.min(dim=1)
        best[c0:c1] = torch.stack([mx, (ix + r.v_off).float(), mn, (jn + r.v_off).float()], dim=1)
        del z, u, zg
    if r.vocab_par:
        allb = torch.empty(r.world, r.T, 4, dtype=torch.float32, device=r.dev)
        dist.all_gather_into_tensor(allb, best)
        k_mx = allb[:, :, 0].argmax(dim=0)
        k_mn = allb[:, :, 2].argmin(dim=0)
        rows = torch.arange(r.T, device=r.dev)
        y, y_min = allb[k_mx, rows, 1], allb[k_mn, rows, 3]
    else:
        y, y_min = best[:, 1], best[:, 3]
    y = torch.where(r.b["spikes"], y_min, y)
    return y.round().to(torch.int32).contiguous()


def _stored_infer_logprobs(r):
    """The stored inference log-probs: the trainer's own log-prob minus the drawn mismatch."""
    import torch
    import torch.distributed as dist

    import paper_2512_16144_b200 as rl

    logp_ref = torch.empty(r.T, dtype=torch.float32, device=r.dev)
    if r.vocab_par:
        parts = torch.empty(r.world, r.T, 4, dtype=torch.float32, device=r.dev)
        ws0 = rl.alloc_workspace(rl.rl_workspace_bytes(r.shape, r.R, 16384), r.dev)
        rl.rl_fwd_partials(r.shape, r.b["hidden"], r.b["w"], r.targets, parts[r.rank], workspace=ws0)
        dist.all_gather_into_tensor(parts, parts[r.rank].contiguous())
        rl.rl_merge_partials(parts, r.world, r.T, logp_ref)
        del ws0
    else:
        rl.rl_logprob_fwd(r.shape, r.b["hidden"], r.b["w"], r.targets, logp_ref)
    infer = torch.clamp(logp_ref - r.b["delta"], max=0.0)
    return torch.where(r.b["spikes"], torch.zeros_like(infer), infer).contiguous()


def _make_engine(r, args):
    """Output buffers, workspace and (N > 1) the multi-GPU engine; returns step()."""
    import torch

    import paper_2512_16144_b200 as rl
    from paper_2512_16144_b200 import parallel

    f32 = dict(dtype=torch.float32, device=r.dev)
    r.phases = parallel.LibrlPhases(dense_backward=args.dense_backward)
    r.adv = torch.empty(r.R, **f32)
    r.report = rl.new_report(r.dev)
    r.logprob = torch.empty(r.T, **f32)
    r.lse = torch.empty(r.T, **f32)
    r.coef = torch.empty(r.T, **f32)
    r.dw = torch.empty(r.V_local, r.H, **f32)
    nv = args.collective == "nvls"
    if r.vocab_par:
        r.engine = parallel.VocabParallelPolicyLoss(r.phases, T=r.T, H=r.H, V_global=r.Vt, num_rollouts=r.R,
                                                    group_size=r.wl_rank.group_size, loss_denominator=r.D,
                                                    dz_chunk_rows=r.chunk, device=r.dev, nvls=nv)
        r.ws, r.dh = r.engine.ws, r.engine.d_hidden
    elif r.world > 1:
        r.engine = parallel.DataParallelPolicyLoss(r.phases, T=r.T, H=r.H, V=r.Vt, num_rollouts=r.R,
                                                   group_size=r.wl_rank.group_size, loss_denominator=r.D,
                                                   device=r.dev, overlap=args.overlap, comm_sms=args.comm_sms,
                                                   nvls=nv, reduce_scatter=args.dw_reduce_scatter and nv)
        r.ws, r.dh = r.engine.ws, r.engine.d_hidden
    else:
        r.engine = None
        r.ws = rl.alloc_workspace(rl.rl_workspace_bytes(r.shape, r.R, r.chunk), r.dev)
        r.dh = torch.empty(r.T, r.H, dtype=torch.bfloat16, device=r.dev)
    torch.cuda.synchronize()
    r.launches = 0
    hidden, w_loc = r.b["hidden"], r.b["w"]

    def step():
        r.phases.launches = 0
        if r.engine is not None:
            r.engine.step(hidden, w_loc, r.targets, r.infer, r.rewards, r.offsets, r.loss_mask, r.dw)
        else:
            r.phases.group_advantages(r.rewards, r.wl_rank.group_size, r.adv)
            r.phases.full_step(r.shape, r.params, hidden, w_loc, r.targets, r.infer, r.adv, r.offsets, r.loss_mask,
                               report=r.report, logprob=r.logprob, lse=r.lse, coef=r.coef, d_hidden=r.dh,
                               d_w_vocab=r.dw, dz_chunk_rows=r.chunk, workspace=r.ws)
        r.launches = r.phases.launches

    return step


def _time_steps(r, args, step):
    """W warm-up steps, then exactly K timed steps between barriers + syncs, CUDA events
    on the launching stream, max over ranks; per-launch kernel times and clocks."""
    import torch
    import torch.distributed as dist

    import paper_2512_16144_b200 as rl

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if r.world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rl.rl_profile_enable(True)
    rl.rl_profile_read()
    with ClockSampler([r.local] if r.world == 1 else list(range(r.world))) as clk:
        torch.cuda.synchronize()
        if r.world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if r.world > 1:
            dist.barrier()
    rl.rl_profile_enable(False)
    r.prof = rl.rl_profile_read(1 << 16)
    r.ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([r.ms], dtype=torch.float64, device=r.dev)
    if r.world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    r.ms_max = float(t.item())
    r.clk = clk
    r.value = (r.T if r.vocab_par else r.T * r.world) / (r.ms_max / 1e3)


def _kernel_report(r, args):
    """Per-kernel shares and rooflines; the roofline object of the dominant kernel."""
    per = {}
    for k, m in r.prof:
        c = per.setdefault(k, [0, 0.0])
        c[0] += 1
        c[1] += m
    kern = {k: {"launches": v[0], "avg_ms": v[1] / v[0], "share": v[1] / (r.ms * args.steps)} for k, v in per.items()}
    # the backward GEMMs run over the rows with coef != 0 (sparse backward, also with
    # the fused NVLS reductions) unless --dense-backward; FLOPs per launch = the step's
    # FLOPs of that kernel / its launches per step
    T, H, V_local = r.T, r.H, r.V_local
    coef_t = r.engine.coef if r.engine is not None else r.coef
    dense = args.dense_backward
    r.kept_rows = int((coef_t != 0).sum().item())
    bwd_rows = T if dense else r.kept_rows
    step_kflops = {"K1_fwd_gemm_lse": 2.0 * T * V_local * H, "K4_bwd_dz_gemm": 2.0 * bwd_rows * V_local * H,
                   "K5_dh_gemm": 2.0 * bwd_rows * V_local * H, "K6_dw_gemm": 2.0 * bwd_rows * V_local * H}
    flops = {k: f / (per[k][0] / args.steps) for k, f in step_kflops.items() if k in per}
    dom = max((k for k in per if k in flops), key=lambda k: per[k][1])
    peaks, peak_src = load_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    burst = float(peaks.get("bf16_tflops", peak))
    achieved = flops[dom] / (kern[dom]["avg_ms"] / 1e3) / 1e12
    # every kernel against its own roofline: the GEMMs in TF/s, the HBM-side kernels in
    # GB/s of algorithmic bytes (K2: the [tiles x T] float4 partials + 3 outputs; the
    # compaction group: gather + scatter of the kept rows, 2 x read+write of n x H bf16)
    hbm_peak = float(peaks.get("hbm_gbs", 6459.3))
    n_tiles = -(-V_local // 256)
    hbm_bytes = {"K2_merge": 16.0 * n_tiles * T + 12.0 * T,
                 "compact": (8.0 * bwd_rows * H + 4.0 * T) if not dense else 0.0,
                 # K4 from K1's probability cache: fp16 p~ read + bf16 dU written per element,
                 # one fp32 m per 32 columns
                 "K4_dz_from_cache": (4.0 + 4.0 / 32) * bwd_rows * V_local}
    for k, v in kern.items():
        if k in flops:
            v["tflops"] = flops[k] / (v["avg_ms"] / 1e3) / 1e12
            v["frac_of_sustained_bf16"] = v["tflops"] / peak
            v["frac_of_burst_bf16"] = v["tflops"] / burst
        elif k in hbm_bytes and hbm_bytes[k] > 0:
            per_launch = hbm_bytes[k] / (v["launches"] / args.steps)
            v["gbs"] = per_launch / (v["avg_ms"] / 1e3) / 1e9
            v["frac_of_hbm"] = v["gbs"] / hbm_peak
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            # measured for the per-rank GLM-16k shape only (profiles/traffic.json)
            # (one GPU, no fused collective: the NVLS epilogue adds its own traffic)
            same = (T, V_local) == (16384, 151552) and r.world == 1
            traffic = json.load(open(tpath)).get(f"{r.name}:{dom}") if same else None
        except Exception:  # noqa: BLE001
            traffic = None
    step_flops = 8.0 * H * V_local * T   # algorithmic 8HV per token on this rank
    rate = lambda f: f / (r.ms_max / 1e3) / 1e12  # noqa: E731
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": f"bf16_tflops_sustained, {peak_src}",
            # the sustained peak is cuBLAS looped for 4 s at its own power-capped clock
            # (MEASURED_PEAKS clocks_under_load); a kernel whose step runs cooler can exceed it
            "peak_burst": burst, "frac_vs_burst": achieved / burst,
            "peak_sm_mhz": (peaks.get("clocks_under_load") or {}).get("sm_mhz_median"),
            "step_frac_8HV": rate(step_flops) / peak,
            "step_frac_8HV_vs_burst": rate(step_flops) / float(peaks.get("bf16_tflops", peak)),
            "step_frac_6HV": rate(0.75 * step_flops) / peak,
            "bwd_rows": bwd_rows,
            # the GEMM FLOPs this step ran (K4 from K1's probability cache runs no GEMM)
            "step_frac_executed": rate(sum(f for k, f in step_kflops.items() if k in per)) / peak}
    return kern, roof


def _timed_host_steps(r, args, hstep):
    """Warm-up, then K host-driven steps on the wall clock (each ends in a D2H read), max over ranks."""
    import torch
    import torch.distributed as dist

    for _ in range(max(1, args.warmup)):
        hstep()
    torch.cuda.synchronize()
    if r.world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        hstep()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / args.steps
    t = torch.tensor([el], dtype=torch.float64, device=r.dev)
    if r.world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _e2e_dp(r, args):
    """e2e through the host-I/O C call (pinned inputs in, report out, every step)."""
    import torch
    import torch.distributed as dist

    import paper_2512_16144_b200 as rl

    b = r.b
    hpin = b["hidden"].view(torch.int16).cpu().pin_memory()
    tpin = r.targets.cpu().pin_memory()
    ipin = r.infer.cpu().pin_memory()
    rpin = torch.from_numpy(b["rewards"]).pin_memory()
    opin = torch.from_numpy(b["offsets"]).pin_memory()
    mpin = torch.from_numpy(b["loss_mask"]).pin_memory()
    r.ws = None                     # the host-I/O call needs its own (larger) workspace
    if r.engine is not None:
        r.engine.ws = None
    wsh = rl.alloc_workspace(rl.rl_workspace_bytes_hostio(r.shape, r.R, r.chunk), r.dev)
    nvls_dp = r.engine is not None and getattr(r.engine, "nvls", None) is not None

    def hstep():
        if nvls_dp:
            rl.rl_policy_loss_fwd_bwd_hostio(r.shape, r.params, r.wl_rank.group_size, hpin, b["w"], tpin, ipin, rpin,
                                             opin, mpin, report=r.report, d_hidden=r.dh, d_w_vocab=r.engine.nvls.buf,
                                             d_w_vocab_nvls=r.engine.nvls.descriptor(
                                                 mode=1 if r.engine.reduce_scatter else 0),
                                             dz_chunk_rows=r.chunk, dense_backward=args.dense_backward,
                                             workspace=wsh)
            r.engine.nvls.barrier()
            return
        rl.rl_policy_loss_fwd_bwd_hostio(r.shape, r.params, r.wl_rank.group_size, hpin, b["w"], tpin, ipin, rpin,
                                         opin, mpin, report=r.report, d_hidden=r.dh, d_w_vocab=r.dw,
                                         dz_chunk_rows=r.chunk, dense_backward=args.dense_backward, workspace=wsh)
        if r.world > 1:
            dist.all_reduce(r.dw)

    el = _timed_host_steps(r, args, hstep)
    T, H, R = r.T, r.H, r.R
    h2d = T * H * 2 + T * 4 + T * 4 + R * 4 + (R + 1) * 4 + T
    return {"value": T * r.world / el, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 48,
            "ms_per_step": el * 1e3, "api": "rl_policy_loss_fwd_bwd_hostio"}


def _e2e_vocab(r, args):
    """Vocab-parallel end to end through VocabParallelPolicyLoss.step_host: every rank
    uploads the (replicated) step inputs from pinned host memory, the hidden rows in
    slabs under the forward, and reads the report back."""
    import torch

    pins = {"hidden": r.b["hidden"].view(torch.int16).cpu().pin_memory(), "targets": r.targets.cpu().pin_memory(),
            "infer": r.infer.cpu().pin_memory(), "rewards": r.rewards.cpu().pin_memory(),
            "offsets": r.offsets.cpu().pin_memory(), "loss_mask": r.loss_mask.cpu().pin_memory()}
    rep_h = torch.empty(48, dtype=torch.uint8).pin_memory()

    def hstep():
        r.engine.step_host(pins["hidden"], r.b["w"], pins["targets"], pins["infer"], pins["rewards"],
                           pins["offsets"], pins["loss_mask"], r.dw)
        rep_h.copy_(r.engine.report, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    el = _timed_host_steps(r, args, hstep)
    return {"value": r.T / el, "unit": "tokens/s",
            "h2d_bytes_per_step": int(sum(v.numel() * v.element_size() for v in pins.values())),
            "d2h_bytes_per_step": 48, "ms_per_step": el * 1e3,
            "api": "parallel.VocabParallelPolicyLoss.step_host (pinned host inputs, per rank)"}


def _config(r, args):
    T, H, V_local, world = r.T, r.H, r.V_local, r.world
    nv = args.collective == "nvls"
    cfg = {"workload": r.name, "T_per_rank": T, "H": H, "V": r.Vt, "V_local": V_local, "rollouts_per_rank": r.R,
           "group_size": r.wl_rank.group_size, "parallelism": f"{r.mode}{world}",
           "l2": "inputs exceed L2 (W %.2f GB, hidden %.0f MB > 126 MB); no flush needed" % (
               V_local * H * 2 / 1e9, T * H * 2 / 1e6),
           "dz_chunk_rows": r.chunk or T,
           "targets": args.targets + (" from the policy (Gumbel-max), guard spikes on the least likely token"
                                      if args.targets == "sampled" else " ids"),
           "kept_row_frac": r.kept_rows / T if T else 0.0,
           "delta_sigma": r.wl_rank.delta_sigma,
           "backward": ("dense" if args.dense_backward else "sparse (rows with coef != 0)") +
                       ("; K4 from K1's probability cache" if any(k == "K4_dz_from_cache" for k, _ in r.prof)
                        else "; K4 recomputes the logits"),
           "collectives": ([] if world == 1 else
                           (["all_gather partials (NCCL)", "dH fp32 all-reduce " +
                             ("fused in K5 epilogue (NVLS multimem)" if nv else "(NCCL)")]
                            if r.vocab_par else
                            ["dW fp32 all-reduce " + ("fused in K6 epilogue (NVLS multimem)" if nv else "(NCCL)")]))}
    if world > 1:
        # the step's exchange and its NVLink roofline (900 GB/s per direction): NVLS moves
        # about 1x the buffer per GPU and direction, a ring all-reduce 2(N-1)/N x
        nb = (T * H * 4) if r.vocab_par else (V_local * H * 4)
        rs = (not r.vocab_par) and args.dw_reduce_scatter and nv
        per_dir = (nb * (world - 1) / world if rs else nb) if nv else 2 * (world - 1) / world * nb
        cfg["collective"] = {"op": ("dH" if r.vocab_par else "dW") + " fp32 " +
                             ("reduce-scatter (vocab rows)" if rs else "all-reduce"),
                             "buffer_bytes": nb, "bytes_per_gpu_per_direction": per_dir,
                             "nvlink_roofline_ms": per_dir / 900e9 * 1e3}
    return cfg


def main_ours(args):
    import torch.distributed as dist

    r = _setup(args)
    if args.targets == "sampled":
        r.targets = r.b["targets"] = _sample_targets(r)
    r.infer = _stored_infer_logprobs(r)
    step = _make_engine(r, args)
    _time_steps(r, args, step)
    kern, roof = _kernel_report(r, args)
    e2e = None
    if not args.no_e2e:
        e2e = _e2e_vocab(r, args) if r.vocab_par else _e2e_dp(r, args)
    clocks = r.clk.summary()
    if roof and clocks.get("sm_mhz"):
        import torch
        # the tcgen05 bound at the clock the step actually ran (median nvidia-smi sample of the
        # timed region): 8192 dense bf16 FLOP per SM clock (the ideal-cycle count of DESIGN.md §5)
        sms = torch.cuda.get_device_properties(r.dev).multi_processor_count
        ideal = sms * 8192.0 * float(clocks["sm_mhz"]) * 1e6 / 1e12
        roof["tensor_ideal_at_sm_clock"] = ideal
        roof["frac_vs_ideal_at_sm_clock"] = roof["achieved"] / ideal
        roof["ideal_note"] = (f"{sms} SMs x 8192 FLOP/clk at the step's median nvidia-smi SM clock (a few samples); "
                              "the clock inside each kernel differs, ncu's cycle counts are the per-kernel figure")
    if r.rank == 0:
        out = {"metric": METRIC, "value": r.value, "unit": "tokens/s", "n_gpus": r.world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": r.ms_max, "higher_is_better": True,
               "scaling": "strong" if r.vocab_par else "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (seeded; GLM-4.5-Air-shaped rollouts, random-init W)", "config": _config(r, args),
               "roofline": roof, "e2e": e2e, "gpu_launches": r.launches * args.steps,
               "clocks": clocks, "kernels": kern, "impl": "ours",
               # the paper prints no number for this path; its whole-system
               # H200 figures, with their hardware, as context only (not a target)
               "context": {"paper_h200": "RL step ~1500 s on 60 nodes x 8 H200 (16 trainer nodes = 128 GPUs), "
                                         "256 prompts x 16 rollouts, <= 64k context: <= 179k tokens/s over the "
                                         "trainer, <= 1.4k per trainer H200, whole model incl. attention and MoE "
                                         "(P:L437-445; BASELINE.md §2)",
                           "vs_baseline": "null: no published number for this metric and workload"}}
        if r.world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(r.wl, budget_s=args.cpu_budget)
        emit(out)
    if r.world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40,
                    help="timed steps (40 x ~60 ms: >= 2 s back to back, so the clock reaches its sustained power-capped state)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=["auto", "small", "glm16k", "glm64k", "stress"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-tokens", type=int, default=0, help="reference arm: tokens per step (0 = 256, or 64 for > 40 steps)")
    ap.add_argument("--dense-backward", action="store_true",
                    help="run the backward GEMMs over all rows instead of the coef != 0 rows (A/B)")
    ap.add_argument("--dw-reduce-scatter", action="store_true",
                    help="DP + NVLS: reduce-scatter dW by vocab rows (FSDP-consistent) instead of all-reduce")
    ap.add_argument("--overlap", action="store_true", help="DP + NCCL: all-reduce dW on a side stream under K5")
    ap.add_argument("--collective", default="auto", choices=["auto", "nccl", "nvls"],
                    help="nvls: the dW (DP) / dH (vocab-parallel) all-reduce is fused into the GEMM epilogue "
                         "over NVLink multicast; auto = nvls when the GPUs support multicast, else NCCL")
    ap.add_argument("--comm-sms", type=int, default=24, help="DP overlap: SMs left to NCCL while K5 runs")
    ap.add_argument("--tokens", type=int, default=0,
                    help="override the workload's tokens per rank (A/B: micro-batch size sweep)")
    ap.add_argument("--dz-chunk", type=int, default=-1,
                    help="rows of the bf16 dU buffer per backward pass (A/B; -1 = auto: T up to 16k rows, else 16k)")
    ap.add_argument("--delta-sigma", type=float, default=None,
                    help="override the workload's log-prob mismatch sigma (A/B: 1.0 = the stress config's)")
    ap.add_argument("--targets", default="sampled", choices=["sampled", "uniform"],
                    help="sampled: y ~ the policy itself (Gumbel-max, guard spikes on the least likely token); "
                         "uniform: uniform ids (round-1 workload)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
