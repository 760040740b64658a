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
def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_16144_b200 as rl
    import synth

    rank, world, local = env_rank()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    name, wl = workload_for(args, world)
    if args.collective == "auto":
        args.collective = "nccl"
        if world > 1:
            import torch.distributed._symmetric_memory as symm_mem
            try:
                probe = symm_mem.empty(1024, dtype=torch.float32, device=dev)
                ok = torch.tensor([1 if symm_mem.rendezvous(probe, dist.group.WORLD.group_name).multicast_ptr
                                   else 0], device=dev)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                args.collective = "nvls" if ok.item() else "nccl"
            except Exception:  # noqa: BLE001 - no symmetric memory / multicast here: NCCL
                args.collective = "nccl"
    vocab_par = name == "glm64k" and world > 1
    mode = "vocab" if vocab_par else "dp"
    H, Vt = wl.hidden, wl.vocab
    if name == "stress":
        # 16k tokens and one G=16 prompt group per rank (the guard and advantages stay local)
        T = wl.tokens // wl.n_ranks
        wl_rank = synth.Workload("stress-rank", 1, wl.group_size, wl.rollout_len, H, Vt,
                                 delta_sigma=wl.delta_sigma, spike_rate=wl.spike_rate)
    else:
        T = wl.tokens
        wl_rank = wl
    if vocab_par:
        assert Vt % world == 0
        V_local, v_off = Vt // world, rank * (Vt // world)
    else:
        V_local, v_off = Vt, 0
    seed = 1000 + (0 if vocab_par else rank)
    b = synth.make_batch_device(wl_rank, seed, device=dev, tokens=T, vocab=V_local, vocab_offset=v_off,
                                vocab_total=Vt)
    R = len(b["offsets"]) - 1
    shape = rl.make_shape(T, H, V_local, v_off, Vt)
    f32 = dict(dtype=torch.float32, device=dev)
    targets = b["targets"]
    offsets = torch.from_numpy(b["offsets"]).to(dev)
    loss_mask = torch.from_numpy(b["loss_mask"]).to(dev)
    rewards = torch.from_numpy(b["rewards"]).to(dev)
    D_local = float(b["loss_mask"].sum())
    if world > 1 and not vocab_par:
        t = torch.tensor([D_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        D = float(t.item())
    else:
        D = D_local
    params = rl.make_params(R, D)

    # stored inference log-probs: the trainer's own log-prob minus the drawn mismatch
    logp_ref = torch.empty(T, **f32)
    if vocab_par:
        parts = torch.empty(world, T, 4, **f32)
        ws0 = rl.alloc_workspace(rl.rl_workspace_bytes(shape, R, 16384), dev)
        rl.rl_fwd_partials(shape, b["hidden"], b["w"], targets, parts[rank], workspace=ws0)
        dist.all_gather_into_tensor(parts, parts[rank].contiguous())
        rl.rl_merge_partials(parts, world, T, logp_ref)
        del ws0
    else:
        rl.rl_logprob_fwd(shape, b["hidden"], b["w"], targets, logp_ref)
    infer = torch.clamp(logp_ref - b["delta"], max=0.0)
    infer = torch.where(b["spikes"], torch.zeros_like(infer), infer).contiguous()
    del logp_ref

    from paper_2512_16144_b200 import parallel
    phases = parallel.LibrlPhases(dense_backward=args.dense_backward)
    adv = torch.empty(R, **f32)
    report = rl.new_report(dev)
    logprob = torch.empty(T, **f32)
    lse = torch.empty(T, **f32)
    coef = torch.empty(T, **f32)
    dw = torch.empty(V_local, H, **f32)
    # dU in 16k-row chunks: keeps K5/K6's per-wave working set inside L2 (the K = T
    # reduction of K6 at 64k rows loses ~20% to HBM re-reads otherwise)
    chunk = 0 if T <= 16384 else 16384
    if vocab_par:
        nv = args.collective == "nvls"
        engine = parallel.VocabParallelPolicyLoss(phases, T=T, H=H, V_global=Vt, num_rollouts=R,
                                                  group_size=wl_rank.group_size, loss_denominator=D,
                                                  dz_chunk_rows=0 if nv else chunk, device=dev, nvls=nv)
        ws = engine.ws
        dh = engine.d_hidden
    elif world > 1:
        engine = parallel.DataParallelPolicyLoss(phases, T=T, H=H, V=Vt, num_rollouts=R,
                                                 group_size=wl_rank.group_size, loss_denominator=D, device=dev,
                                                 overlap=args.overlap, comm_sms=args.comm_sms,
                                                 nvls=args.collective == "nvls",
                                                 reduce_scatter=args.dw_reduce_scatter and args.collective == "nvls")
        ws = engine.ws
        dh = engine.d_hidden
    else:
        engine = None
        ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, R, chunk), dev)
        dh = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()

    launches = [0]
    hidden, w_loc = b["hidden"], b["w"]

    def step():
        phases.launches = 0
        if engine is not None:
            engine.step(hidden, w_loc, targets, infer, rewards, offsets, loss_mask, dw)
        else:
            phases.group_advantages(rewards, wl_rank.group_size, adv)
            phases.full_step(shape, params, hidden, w_loc, targets, infer, adv, offsets, loss_mask, report=report,
                             logprob=logprob, lse=lse, coef=coef, d_hidden=dh, d_w_vocab=dw, dz_chunk_rows=chunk,
                             workspace=ws)
        launches[0] = phases.launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rl.rl_profile_enable(True)
    rl.rl_profile_read()
    with ClockSampler([local] if world == 1 else list(range(world))) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    rl.rl_profile_enable(False)
    prof = rl.rl_profile_read(1 << 16)
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    tokens_per_step = T if vocab_par else T * world
    value = tokens_per_step / (ms_max / 1e3)

    # per-kernel share of the timed region and the dominant kernel's roofline
    per = {}
    for k, m in prof:
        c = per.setdefault(k, [0, 0.0])
        c[0] += 1
        c[1] += m
    total_k = sum(v[1] for v in per.values())
    kern = {k: {"launches": v[0], "avg_ms": v[1] / v[0], "share": v[1] / (ms * args.steps)} for k, v in per.items()}
    # the backward GEMMs run over the rows with coef != 0 (sparse backward) unless the
    # vocab-parallel NVLS dH reduction forces the dense path; FLOPs per launch = the
    # step's FLOPs of that kernel / its launches per step
    coef_t = engine.coef if engine is not None else coef
    dense = args.dense_backward or (vocab_par and args.collective == "nvls")
    bwd_rows = T if dense else int((coef_t != 0).sum().item())
    step_kflops = {"K1_fwd_gemm_lse": 2.0 * T * V_local * H, "K4_bwd_dz_gemm": 2.0 * bwd_rows * V_local * H,
                   "K5_dh_gemm": 2.0 * bwd_rows * V_local * H, "K6_dw_gemm": 2.0 * bwd_rows * V_local * H}
    flops = {k: f / (per[k][0] / args.steps) for k, f in step_kflops.items() if k in per}
    dom = max((k for k in per if k in flops), key=lambda k: per[k][1])
    peaks, peak_src = load_peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    achieved = flops[dom] / (kern[dom]["avg_ms"] / 1e3) / 1e12
    # every kernel against its own roofline: the GEMMs in TF/s, the HBM-side kernels in
    # GB/s of algorithmic bytes (K2: the [tiles x T] float4 partials + 3 outputs; the
    # compaction group: gather + scatter of the kept rows, 2 x read+write of n x H bf16)
    hbm_peak = float(peaks.get("hbm_gbs", 6459.3))
    n_tiles = -(-V_local // 256)
    hbm_bytes = {"K2_merge": 16.0 * n_tiles * T + 12.0 * T,
                 "compact": (8.0 * bwd_rows * H + 4.0 * T) if not dense else 0.0}
    for k, v in kern.items():
        if k in flops:
            v["tflops"] = flops[k] / (v["avg_ms"] / 1e3) / 1e12
            v["frac_of_sustained_bf16"] = v["tflops"] / peak
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
            same = (T, V_local) == (16384, 151552) and world == 1
            traffic = json.load(open(tpath)).get(f"{name}:{dom}") if same else None
        except Exception:
            traffic = None
    step_flops = 8.0 * H * V_local * T   # algorithmic 8HV per token on this rank
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": f"bf16_tflops_sustained, {peak_src}",
            "step_frac_8HV": (step_flops / (ms_max / 1e3) / 1e12) / peak,
            "step_frac_8HV_vs_burst": (step_flops / (ms_max / 1e3) / 1e12) / float(peaks.get("bf16_tflops", peak)),
            "step_frac_6HV": (0.75 * step_flops / (ms_max / 1e3) / 1e12) / peak,
            "bwd_rows": bwd_rows,
            "step_frac_executed": (sum(step_kflops.values()) / (ms_max / 1e3) / 1e12) / peak}

    # e2e through the host-I/O C call (pinned inputs in, report out, every step)
    e2e = None
    if not vocab_par and not args.no_e2e:
        hpin = b["hidden"].view(torch.int16).cpu().pin_memory()
        tpin = targets.cpu().pin_memory()
        ipin = infer.cpu().pin_memory()
        rpin = torch.from_numpy(b["rewards"]).pin_memory()
        opin = torch.from_numpy(b["offsets"]).pin_memory()
        mpin = torch.from_numpy(b["loss_mask"]).pin_memory()
        del ws
        if engine is not None:
            engine.ws = None
        wsh = rl.alloc_workspace(rl.rl_workspace_bytes_hostio(shape, R, chunk), dev)

        nvls_dp = engine is not None and getattr(engine, "nvls", None) is not None

        def hstep():
            if nvls_dp:
                rl.rl_policy_loss_fwd_bwd_hostio(shape, params, wl_rank.group_size, hpin, b["w"], tpin, ipin, rpin,
                                                 opin, mpin, report=report, d_hidden=dh, d_w_vocab=engine.nvls.buf,
                                                 d_w_vocab_nvls=engine.nvls.descriptor(
                                                     mode=1 if engine.reduce_scatter else 0),
                                                 dz_chunk_rows=chunk,
                                                 dense_backward=args.dense_backward, workspace=wsh)
                engine.nvls.barrier()
                return
            rl.rl_policy_loss_fwd_bwd_hostio(shape, params, wl_rank.group_size, hpin, b["w"], tpin, ipin, rpin, opin,
                                             mpin, report=report, d_hidden=dh, d_w_vocab=dw, dz_chunk_rows=chunk,
                                             dense_backward=args.dense_backward, workspace=wsh)
            if world > 1:
                dist.all_reduce(dw)

        for _ in range(max(1, args.warmup)):
            hstep()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hstep()
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / args.steps
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
        h2d = T * H * 2 + T * 4 + T * 4 + R * 4 + (R + 1) * 4 + T
        e2e = {"value": T * world / el, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 48,
               "ms_per_step": el * 1e3, "api": "rl_policy_loss_fwd_bwd_hostio"}
    elif vocab_par and not args.no_e2e:
        # vocab-parallel end to end: every rank uploads the (replicated) step inputs from
        # pinned host memory, runs the split-phase engine and reads the report back
        pins = {"hidden": b["hidden"].cpu().pin_memory(), "targets": targets.cpu().pin_memory(),
                "infer": infer.cpu().pin_memory(), "rewards": rewards.cpu().pin_memory(),
                "offsets": offsets.cpu().pin_memory(), "loss_mask": loss_mask.cpu().pin_memory()}
        devs = {k: torch.empty_like(v, device=dev) for k, v in pins.items()}
        rep_h = torch.empty(48, dtype=torch.uint8).pin_memory()

        def hstep():
            for k, v in pins.items():
                devs[k].copy_(v, non_blocking=True)
            engine.step(devs["hidden"], w_loc, devs["targets"], devs["infer"], devs["rewards"], devs["offsets"],
                        devs["loss_mask"], dw)
            rep_h.copy_(engine.report, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(max(1, args.warmup)):
            hstep()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hstep()
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / args.steps
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
        e2e = {"value": T / el, "unit": "tokens/s",
               "h2d_bytes_per_step": int(sum(v.numel() * v.element_size() for v in pins.values())),
               "d2h_bytes_per_step": 48, "ms_per_step": el * 1e3,
               "api": "parallel.VocabParallelPolicyLoss.step (host inputs, per rank)"}

    out = None
    if rank == 0:
        cfg = {"workload": name, "T_per_rank": T, "H": H, "V": Vt, "V_local": V_local, "rollouts_per_rank": R,
               "group_size": wl_rank.group_size, "parallelism": f"{mode}{world}",
               "l2": "inputs exceed L2 (W %.2f GB, hidden %.0f MB > 126 MB); no flush needed" % (
                   V_local * H * 2 / 1e9, T * H * 2 / 1e6),
               "dz_chunk_rows": (T if (vocab_par and args.collective == "nvls") else (chunk or T)),
               "collectives": ([] if world == 1 else
                               (["all_gather partials (NCCL)", "dH fp32 all-reduce " +
                                 ("fused in K5 epilogue (NVLS multimem)" if args.collective == "nvls" else "(NCCL)")]
                                if vocab_par else
                                ["dW fp32 all-reduce " + ("fused in K6 epilogue (NVLS multimem)"
                                                          if args.collective == "nvls" else "(NCCL)")]))}
        if world > 1:
            # the step's exchange and its NVLink roofline (900 GB/s per direction): NVLS moves
            # about 1x the buffer per GPU and direction, a ring all-reduce 2(N-1)/N x
            nb = (T * H * 4) if vocab_par else (V_local * H * 4)
            rs = (not vocab_par) and args.dw_reduce_scatter and args.collective == "nvls"
            per_dir = (nb * (world - 1) / world if rs else nb) if args.collective == "nvls" \
                else 2 * (world - 1) / world * nb
            cfg["collective"] = {"op": ("dH" if vocab_par else "dW") + " fp32 " +
                                 ("reduce-scatter (vocab rows)" if rs else "all-reduce"),
                                 "buffer_bytes": nb, "bytes_per_gpu_per_direction": per_dir,
                                 "nvlink_roofline_ms": per_dir / 900e9 * 1e3}
        out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
               "scaling": "strong" if vocab_par else "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (seeded; GLM-4.5-Air-shaped rollouts, random-init W)", "config": cfg,
               "roofline": roof, "e2e": e2e, "gpu_launches": launches[0] * args.steps,
               "clocks": clk.summary(), "kernels": kern, "impl": "ours"}
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(wl, budget_s=args.cpu_budget)
        emit(out)
    if world > 1:
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
