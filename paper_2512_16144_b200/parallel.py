"""Multi-GPU composition of the step: one process per GPU,
torch.distributed process groups (NCCL over NVLink) for the collectives, librl's
split-phase C calls for all arithmetic.

* DataParallelPolicyLoss — each rank runs the whole step on its own rollouts
  (whole groups per rank, so the guard and the advantages stay local) with the
  GLOBAL loss denominator D (reading R5); the exchange step is the dW all-reduce.
* VocabParallelPolicyLoss — W row-sharded; K1 partials (16 B/token) are
  all-gathered and merged in rank order; S3 runs redundantly; the dH partials
  are all-reduced; each rank keeps its complete dW shard.
* SplitRolloutPolicyLoss — data parallel over ANY split of the packed rows, so a
  rollout may straddle ranks (CP-style): the guard's per-rollout min
  ratio is all-reduced (MIN), GSPO's log-ratio sums and counts (SUM); advantages
  come from the whole groups' rewards; dW is all-reduced.

The arithmetic goes through a `phases` object with librl's split-phase
signatures. `LibrlPhases` (the C ABI) is the only implementation in the
package; tests substitute a CPU double to check this host logic on gloo.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import (RL_BWD_ALL, RL_BWD_DENSE, RL_BWD_DH, RL_BWD_DU, RL_BWD_DW, alloc_workspace, make_params,
               make_shape, rl_bwd_ex, rl_fwd_partials, rl_fwd_partials_ex, RL_FWD_CACHE, RL_BWD_FROM_CACHE,
               rl_group_advantages, rl_last_launch_count, rl_logprob_fwd, rl_loss_coef,
               rl_loss_coef_ex, rl_rollout_stats,
               rl_merge_partials, rl_ns_shard_apply, rl_ns_shard_gram, rl_ns_shard_sumsq,
               rl_nvls_flag_count, rl_nvls_reduce, rl_nvls_shard_rows, rl_policy_loss_fwd_bwd, rl_workspace_bytes)


class NvlsReduction:
    """A symmetric fp32 output buffer plus per-slab flags for librl's in-epilogue
    NVLink-multicast all-reduce (rl_nvls_reduce), on torch symmetric memory.

    Each call uses a fresh epoch; `barrier()` (on the current stream) completes the
    exchange: after it every rank's `buf` holds the sum over ranks."""

    def __init__(self, rows, cols, flag_count, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem
        name = (group or dist.group.WORLD).group_name
        self.buf = symm_mem.empty(rows, cols, dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.buf, name)
        if not self.handle.multicast_ptr:
            raise RuntimeError("NVLink multicast (NVLS) is not available for this group")
        self.flags = symm_mem.empty(max(1, flag_count), dtype=torch.int32, device=device)
        self.flags.zero_()
        self.flag_handle = symm_mem.rendezvous(self.flags, name)
        self.rank, self.world = self.handle.rank, self.handle.world_size
        self.epoch = 0
        torch.cuda.synchronize(device)
        self.handle.barrier(channel=0)

    def descriptor(self, lag=None, mode=0) -> rl_nvls_reduce:
        """lag: 0 (default, RL_NVLS_LAG) = the GEMM's communication warps reduce each
        slab as soon as every rank published it; > 0 = the epilogue warps reduce the
        slab stored `lag` tiles earlier (the round-1 schedule, for A/B runs)."""
        if lag is None:
            lag = int(os.environ.get("RL_NVLS_LAG", "0"))
        self.epoch += 1
        d = rl_nvls_reduce()
        d.multicast = self.handle.multicast_ptr
        for r in range(self.world):
            d.flags[r] = self.flag_handle.buffer_ptrs[r]
        d.rank, d.world, d.epoch, d.lag, d.mode = self.rank, self.world, self.epoch, lag, mode
        return d

    def barrier(self):
        self.handle.barrier(channel=1)


class LibrlPhases:
    """The split phases backed by librl (device tensors, current stream).
    `dense_backward` runs the backward GEMMs over all rows (RL_BWD_DENSE) instead of
    the rows with a non-zero coefficient."""

    supports_cache = True   # fwd_partials(cache=True) + bwd(from_cache=True): K4 from K1's probability cache

    def __init__(self, dense_backward: bool = False):
        self.launches = 0
        self.dense = RL_BWD_DENSE if dense_backward else 0

    def _count(self):
        self.launches += rl_last_launch_count()

    def group_advantages(self, rewards, group_size, adv):
        rl_group_advantages(rewards, group_size, adv)
        self._count()

    # row-sharded Newton-Schulz (newton_schulz_row_sharded)
    def ns_sumsq(self, g, sumsq, workspace):
        rl_ns_shard_sumsq(g, sumsq, workspace)
        self._count()

    def ns_gram(self, j, g, sumsq, gram, workspace):
        rl_ns_shard_gram(j, g, sumsq, gram, workspace)
        self._count()

    def ns_apply(self, j, steps, gram, M_local, N, out, workspace):
        rl_ns_shard_apply(j, steps, gram, M_local, N, out, workspace)
        self._count()

    def fwd_partials(self, shape, hidden, w_shard, targets, partials, workspace=None, cache=False):
        if cache:   # also fill the probability cache for bwd(..., from_cache=True) on the same workspace
            rl_fwd_partials_ex(shape, hidden, w_shard, targets, partials, RL_FWD_CACHE, workspace=workspace)
        else:
            rl_fwd_partials(shape, hidden, w_shard, targets, partials, workspace=workspace)
        self._count()

    def merge_partials(self, parts, n_parts, T, logprob, entropy, lse):
        rl_merge_partials(parts, n_parts, T, logprob, entropy, lse)
        self._count()

    def loss_coef(self, params, T, V_global, logprob, infer, targets, adv, offsets, loss_mask, coef, keep, guarded,
                  report, workspace=None):
        rl_loss_coef(params, T, V_global, logprob, infer, targets, adv, offsets, loss_mask, coef, keep, guarded,
                     report=report, workspace=workspace)
        self._count()

    def rollout_stats(self, params, T, V_global, logprob, infer, targets, offsets, loss_mask, kmin, logratio_sum,
                      n_valid):
        rl_rollout_stats(params, T, V_global, logprob, infer, targets, offsets, loss_mask, kmin, logratio_sum,
                         n_valid)
        self._count()

    def loss_coef_ex(self, params, T, V_global, logprob, infer, targets, adv, offsets, loss_mask, kmin, logratio_sum,
                     n_valid, coef, keep, guarded, report, workspace=None):
        rl_loss_coef_ex(params, T, V_global, logprob, infer, targets, adv, offsets, loss_mask, kmin, logratio_sum,
                        n_valid, coef, keep, guarded, report=report, workspace=workspace)
        self._count()

    def bwd(self, shape, hidden, w_shard, targets, lse, coef, d_hidden_f32, d_w_vocab, dz_chunk_rows=0,
            workspace=None, dh_nvls=None, from_cache=False):
        rl_bwd_ex(shape, hidden, w_shard, targets, lse, coef, d_hidden_f32=d_hidden_f32, d_w_vocab=d_w_vocab,
                  dz_chunk_rows=dz_chunk_rows,
                  phases=RL_BWD_ALL | self.dense | (RL_BWD_FROM_CACHE if from_cache else 0), dh_nvls=dh_nvls,
                  workspace=workspace)
        self._count()

    def logprob_fwd(self, shape, hidden, w, targets, logprob, entropy, lse, workspace=None):
        rl_logprob_fwd(shape, hidden, w, targets, logprob, entropy, lse, workspace=workspace)
        self._count()

    def bwd_phases(self, shape, hidden, w, targets, lse, coef, d_hidden, d_w_vocab, phases, max_sms=0,
                   workspace=None):
        rl_bwd_ex(shape, hidden, w, targets, lse, coef, d_hidden=d_hidden, d_w_vocab=d_w_vocab,
                  phases=phases | self.dense, max_sms=max_sms, workspace=workspace)
        self._count()

    def full_step(self, shape, params, hidden, w, targets, infer, adv, offsets, loss_mask, *, report, logprob,
                  entropy=None, lse=None, coef=None, keep=None, guarded=None, d_hidden=None, d_w_vocab=None,
                  d_w_vocab_nvls=None, dz_chunk_rows=0, workspace=None, accumulate_dw=False):
        rl_policy_loss_fwd_bwd(shape, params, hidden, w, targets, infer, adv, offsets, loss_mask, report=report,
                               logprob=logprob, entropy=entropy, lse=lse, coef=coef, token_keep=keep,
                               rollout_guarded=guarded, d_hidden=d_hidden, d_w_vocab=d_w_vocab,
                               d_w_vocab_nvls=d_w_vocab_nvls, dz_chunk_rows=dz_chunk_rows,
                               dense_backward=bool(self.dense), workspace=workspace, accumulate_dw=accumulate_dw)
        self._count()


def prob_cache_enabled() -> bool:
    """librl's RL_P_CACHE knob (default on): the split phases use the cache only when the
    workspace layout has one."""
    import os
    return os.environ.get("RL_P_CACHE", "1") != "0"


def _all_gather_rows(parts: torch.Tensor, mine: torch.Tensor, group=None):
    """parts[world, ...] <- every rank's `mine`, in rank order."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(parts, mine.contiguous(), group=group)
    else:
        dist.all_gather(list(parts.unbind(0)), mine.contiguous(), group=group)


class VocabParallelPolicyLoss:
    """S0..S6 with W_vocab row-sharded across the ranks of `group`."""

    def __init__(self, phases, *, T, H, V_global, num_rollouts, group_size, loss_denominator, group=None,
                 inv_temperature=1.0, alpha=0.5, beta=5.0, guard=1e-5, dz_chunk_rows=0, device=None,
                 workspace=True, nvls=False, variant="icepop", kl_tau=0.0, kl_set="masked",
                 inv_temperature_rows=None):
        self.ph = phases
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if V_global % self.world:
            raise ValueError("V_global must divide evenly across the vocab-parallel ranks")
        self.V_local = V_global // self.world
        self.vocab_offset = self.rank * self.V_local
        self.T, self.H, self.V_global, self.R, self.G = T, H, V_global, num_rollouts, group_size
        self.invt_rows = inv_temperature_rows          # kept alive: the shape points at it
        self.shape = make_shape(T, H, self.V_local, self.vocab_offset, V_global, inv_temperature,
                                inv_temperature_rows=inv_temperature_rows)
        self.params = make_params(num_rollouts, loss_denominator, alpha, beta, guard, variant, kl_tau, kl_set)
        self.chunk = dz_chunk_rows
        dev = device
        f32 = dict(dtype=torch.float32, device=dev)
        self.parts = torch.empty(self.world, T, 4, **f32)
        self.logprob = torch.empty(T, **f32)
        self.entropy = torch.empty(T, **f32)
        self.lse = torch.empty(T, **f32)
        self.coef = torch.empty(T, **f32)
        self.keep = torch.empty(T, dtype=torch.uint8, device=dev)
        self.guarded = torch.empty(num_rollouts, dtype=torch.uint8, device=dev)
        self.adv = torch.empty(num_rollouts, **f32)
        self.report = torch.zeros(48, dtype=torch.uint8, device=dev)
        # nvls: dH partials are all-reduced inside the K5 epilogue (NVLink multicast),
        # chunk by chunk, over all rows (dense) or the compacted rows (sparse backward)
        self.nvls = None
        if nvls:
            self.nvls = NvlsReduction(T, H, rl_nvls_flag_count(self.shape, 1), group, dev)
            self.d_hidden = self.nvls.buf
        else:
            self.d_hidden = torch.empty(T, H, **f32)
        self.ws = self.loss_ws = None
        if workspace:
            self.ws = alloc_workspace(rl_workspace_bytes(self.shape, num_rollouts, dz_chunk_rows), dev)
            self.loss_ws = alloc_workspace(48 * max(1, num_rollouts), dev)

    def step(self, hidden, w_shard, targets, infer, rewards, offsets, loss_mask, d_w_vocab):
        ph = self.ph
        ph.group_advantages(rewards, self.G, self.adv)
        # the probability cache lives in this engine's workspace from the forward to the backward
        cache = self.ws is not None and getattr(ph, "supports_cache", False) and prob_cache_enabled()
        if cache:
            ph.fwd_partials(self.shape, hidden, w_shard, targets, self.parts[self.rank], workspace=self.ws,
                            cache=True)
        else:
            ph.fwd_partials(self.shape, hidden, w_shard, targets, self.parts[self.rank], workspace=self.ws)
        _all_gather_rows(self.parts, self.parts[self.rank], self.group)                 # exchange 1
        ph.merge_partials(self.parts, self.world, self.T, self.logprob, self.entropy, self.lse)
        ph.loss_coef(self.params, self.T, self.V_global, self.logprob, infer, targets, self.adv, offsets,
                     loss_mask, self.coef, self.keep, self.guarded, self.report, workspace=self.loss_ws)
        kw = {"from_cache": True} if cache else {}
        if self.nvls is not None:
            ph.bwd(self.shape, hidden, w_shard, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
                   dz_chunk_rows=self.chunk, workspace=self.ws, dh_nvls=self.nvls.descriptor(), **kw)
            self.nvls.barrier()                                   # exchange 2, fused into K5's epilogue
            return self.d_hidden
        ph.bwd(self.shape, hidden, w_shard, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
               dz_chunk_rows=self.chunk, workspace=self.ws, **kw)
        dist.all_reduce(self.d_hidden, group=self.group)                                  # exchange 2
        return self.d_hidden

    def step_host(self, hidden_host, w_shard, targets_host, infer_host, rewards_host, offsets_host,
                  loss_mask_host, d_w_vocab, slab_ends=None):
        """step() with the per-step inputs in pinned HOST memory: the small inputs, then the
        hidden rows in slabs, go up on a copy stream, and the forward partials run slab by
        slab as the rows arrive (each row's partial is independent), so the upload hides
        under K1. Returns d_hidden like step().

        The copies are asynchronous: the host buffers must not be modified until
        `self.upload_done` (a CUDA event recorded after the last copy) has completed,
        e.g. `self.upload_done.synchronize()` before refilling them for the next step."""
        dev = w_shard.device
        if getattr(self, "_host_in", None) is None:
            self._host_in = {"hidden": torch.empty(self.T, self.H, dtype=torch.bfloat16, device=dev),
                             "targets": torch.empty(self.T, dtype=torch.int32, device=dev),
                             "infer": torch.empty(self.T, dtype=torch.float32, device=dev),
                             "rewards": torch.empty(self.R, dtype=torch.float32, device=dev),
                             "offsets": torch.empty(self.R + 1, dtype=torch.int32, device=dev),
                             "loss_mask": torch.empty(self.T, dtype=torch.uint8, device=dev)}
            self._copy = torch.cuda.Stream(device=dev)
        d = self._host_in
        ends = slab_ends or [e for e in (1024, 4096) if e < self.T] + list(range(8192, self.T, 8192)) + [self.T]
        main = torch.cuda.current_stream(dev)
        self._copy.wait_stream(main)                      # the previous step is done with the inputs
        small_ev = torch.cuda.Event()
        slab_evs = []
        with torch.cuda.stream(self._copy):
            for k, v in (("targets", targets_host), ("infer", infer_host), ("rewards", rewards_host),
                         ("offsets", offsets_host), ("loss_mask", loss_mask_host)):
                d[k].copy_(v, non_blocking=True)
            small_ev.record()
            r0 = 0
            hidden_view = d["hidden"].view(hidden_host.dtype)
            for r1 in ends:
                hidden_view[r0:r1].copy_(hidden_host[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                slab_evs.append((r0, r1, ev))
                r0 = r1
            self.upload_done = slab_evs[-1][2] if slab_evs else small_ev
        ph = self.ph
        main.wait_event(small_ev)
        ph.group_advantages(d["rewards"], self.G, self.adv)
        mine = self.parts[self.rank]
        for r0, r1, ev in slab_evs:                        # K1 (+ its one-partial-per-row merge) per slab
            main.wait_event(ev)
            sub = make_shape(r1 - r0, self.H, self.V_local, self.vocab_offset, self.V_global,
                             self.shape.inv_temperature,
                             inv_temperature_rows=None if self.invt_rows is None else self.invt_rows[r0:r1])
            ph.fwd_partials(sub, d["hidden"][r0:r1], w_shard, d["targets"][r0:r1], mine[r0:r1], workspace=self.ws)
        _all_gather_rows(self.parts, mine, self.group)                                    # exchange 1
        ph.merge_partials(self.parts, self.world, self.T, self.logprob, self.entropy, self.lse)
        ph.loss_coef(self.params, self.T, self.V_global, self.logprob, d["infer"], d["targets"], self.adv,
                     d["offsets"], d["loss_mask"], self.coef, self.keep, self.guarded, self.report,
                     workspace=self.loss_ws)
        hidden, targets = d["hidden"], d["targets"]
        if self.nvls is not None:
            ph.bwd(self.shape, hidden, w_shard, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
                   dz_chunk_rows=self.chunk, workspace=self.ws, dh_nvls=self.nvls.descriptor())
            self.nvls.barrier()
            return self.d_hidden
        ph.bwd(self.shape, hidden, w_shard, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
               dz_chunk_rows=self.chunk, workspace=self.ws)
        dist.all_reduce(self.d_hidden, group=self.group)
        return self.d_hidden


class DataParallelPolicyLoss:
    """S0..S6 on each rank's own rollouts; dW summed over the ranks of `group`."""

    def __init__(self, phases, *, T, H, V, num_rollouts, group_size, loss_denominator, group=None,
                 inv_temperature=1.0, alpha=0.5, beta=5.0, guard=1e-5, device=None, d_hidden_dtype=torch.bfloat16,
                 workspace=True, overlap=False, comm_sms=24, nvls=False, variant="icepop", kl_tau=0.0,
                 kl_set="masked", inv_temperature_rows=None, reduce_scatter=False, dz_chunk_rows=0):
        self.ph = phases
        self.chunk = dz_chunk_rows
        # overlap: the dW all-reduce (NCCL, side stream) runs concurrently with K5,
        # which then uses all but `comm_sms` SMs (NCCL's NVLS channels need SMs).
        self.overlap = overlap
        self.comm = torch.cuda.Stream(device=device) if overlap else None
        if overlap:
            n_sms = torch.cuda.get_device_properties(device).multi_processor_count
            self.dh_sms = max(2, (n_sms - comm_sms) // 2 * 2)
        self.group = group
        self.world = dist.get_world_size(group)
        self.T, self.H, self.V, self.R, self.G = T, H, V, num_rollouts, group_size
        self.invt_rows = inv_temperature_rows          # kept alive: the shape points at it
        self.shape = make_shape(T, H, V, 0, V, inv_temperature, inv_temperature_rows=inv_temperature_rows)
        self.params = make_params(num_rollouts, loss_denominator, alpha, beta, guard, variant, kl_tau, kl_set)
        dev = device
        f32 = dict(dtype=torch.float32, device=dev)
        self.logprob = torch.empty(T, **f32)
        self.entropy = torch.empty(T, **f32)
        self.lse = torch.empty(T, **f32)
        self.coef = torch.empty(T, **f32)
        self.keep = torch.empty(T, dtype=torch.uint8, device=dev)
        self.guarded = torch.empty(num_rollouts, dtype=torch.uint8, device=dev)
        self.adv = torch.empty(num_rollouts, **f32)
        self.report = torch.zeros(48, dtype=torch.uint8, device=dev)
        self.d_hidden = torch.empty(T, H, dtype=d_hidden_dtype, device=dev)
        self.ws = (alloc_workspace(rl_workspace_bytes(self.shape, num_rollouts, dz_chunk_rows), dev) if workspace
                   else None)
        self.loss_ws = alloc_workspace(48 * max(1, num_rollouts), dev) if workspace else None
        # nvls: dW is all-reduced inside the K6 epilogue (NVLink multicast); the
        # step then returns the symmetric buffer that holds the sum.
        self.nvls = NvlsReduction(V, H, rl_nvls_flag_count(self.shape, 0), group, dev) if nvls else None
        # reduce_scatter (NVLS only, FSDP-consistent): rank r ends with the summed dW rows
        # [r S, (r+1) S) (S = rl_nvls_shard_rows); step() returns that shard
        self.reduce_scatter = bool(reduce_scatter)
        if self.reduce_scatter and not nvls:
            raise ValueError("reduce_scatter needs nvls=True")
        self.shard_rows = rl_nvls_shard_rows(V, self.world) if self.reduce_scatter else None

    @staticmethod
    def global_denominator(loss_mask: torch.Tensor, group=None) -> float:
        """D = sum over ranks of the local loss-token counts (one all-reduce at batch assembly)."""
        t = loss_mask.to(torch.float64).sum().reshape(1)
        dist.all_reduce(t, group=group)
        return float(t.item())

    def step(self, hidden, w, targets, infer, rewards, offsets, loss_mask, d_w_vocab=None, *, accumulate=False,
             reduce=True):
        """One micro-batch. Gradient accumulation over micro-batches (the paper's FSDP
        trainer): pass accumulate=True on all but the first and reduce=False on all
        but the last; dW is summed locally and reduced once, on the last micro-batch
        (fused into its dW GEMM with NVLS). Every micro-batch has this engine's T rows
        and rollouts; D is the global count of loss tokens of the whole step (R5)."""
        ph = self.ph
        ph.group_advantages(rewards, self.G, self.adv)
        if self.nvls is not None:
            ph.full_step(self.shape, self.params, hidden, w, targets, infer, self.adv, offsets, loss_mask,
                         report=self.report, logprob=self.logprob, entropy=self.entropy, lse=self.lse,
                         coef=self.coef, keep=self.keep, guarded=self.guarded, d_hidden=self.d_hidden,
                         d_w_vocab=self.nvls.buf,
                         d_w_vocab_nvls=(self.nvls.descriptor(mode=1 if self.reduce_scatter else 0)
                                         if reduce else None),
                         dz_chunk_rows=self.chunk, workspace=self.ws, accumulate_dw=accumulate)
            if not reduce:
                return self.nvls.buf                              # this rank's partial sum so far
            self.nvls.barrier()                                   # the exchange, fused into K6's epilogue
            if self.reduce_scatter:
                r = dist.get_rank(self.group)
                return self.nvls.buf[r * self.shard_rows:(r + 1) * self.shard_rows]
            return self.nvls.buf
        if not self.overlap or accumulate or not reduce:
            ph.full_step(self.shape, self.params, hidden, w, targets, infer, self.adv, offsets, loss_mask,
                         report=self.report, logprob=self.logprob, entropy=self.entropy, lse=self.lse,
                         coef=self.coef, keep=self.keep, guarded=self.guarded, d_hidden=self.d_hidden,
                         d_w_vocab=d_w_vocab, dz_chunk_rows=self.chunk, workspace=self.ws, accumulate_dw=accumulate)
            if reduce:
                dist.all_reduce(d_w_vocab, group=self.group)                              # the exchange
            return d_w_vocab
        # S1..S3, then K4 (dU) and K6 (dW); the dW all-reduce runs on a side stream
        # while K5 (dH) uses the SMs NCCL leaves free.
        ph.logprob_fwd(self.shape, hidden, w, targets, self.logprob, self.entropy, self.lse, workspace=self.ws)
        ph.loss_coef(self.params, self.T, self.V, self.logprob, infer, targets, self.adv, offsets, loss_mask,
                     self.coef, self.keep, self.guarded, self.report, workspace=self.loss_ws)
        ph.bwd_phases(self.shape, hidden, w, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
                      RL_BWD_DU | RL_BWD_DW, workspace=self.ws)
        main = torch.cuda.current_stream()
        self.comm.wait_stream(main)
        with torch.cuda.stream(self.comm):
            dist.all_reduce(d_w_vocab, group=self.group)                                  # the exchange
        ph.bwd_phases(self.shape, hidden, w, targets, self.lse, self.coef, self.d_hidden, d_w_vocab, RL_BWD_DH,
                      max_sms=self.dh_sms, workspace=self.ws)
        main.wait_stream(self.comm)
        return d_w_vocab


class SplitRolloutPolicyLoss:
    """Data parallel over an arbitrary split of the packed rows (sequence
    sharding): rank r holds rows [row_start, row_start + T) of the global batch whose
    rollouts are `global_offsets` ([R_global + 1], host), so the first and last rollouts
    of a rank may continue on its neighbours. What couples the ranks, besides the dW
    all-reduce:
      * the guard is a min over the WHOLE rollout: per-rollout min ratios of
        every rank are all-reduced (MIN) over [R_global] floats before S3;
      * GSPO's sequence ratio (R17) needs the whole rollout's log-ratio sum and token
        count (SUM over [R_global]);
      * advantages use whole groups: every rank computes them from all
        R_global rewards (a few hundred floats) and keeps its rollouts' slice;
      * D (R5) is the global count of loss tokens.
    Loss values add up over ranks (a split GSPO rollout contributes n_local / n of its
    term on each rank); report.guarded_rollouts is per rank (split rollouts count on
    every rank that holds part of them) — `guarded_global` is the exact count."""

    def __init__(self, phases, *, T, H, V, global_offsets, row_start, group_size, loss_denominator, group=None,
                 inv_temperature=1.0, alpha=0.5, beta=5.0, guard=1e-5, variant="icepop", kl_tau=0.0,
                 kl_set="masked", device=None, d_hidden_dtype=torch.bfloat16, workspace=True, dz_chunk_rows=0):
        import numpy as np
        self.ph = phases
        self.group = group
        self.T, self.H, self.V, self.G = T, H, V, group_size
        off = np.asarray(global_offsets, dtype=np.int64)
        self.R_global = len(off) - 1
        lo, hi = int(row_start), int(row_start) + T
        # the global rollouts with at least one row in [lo, hi) (empty rollouts at the
        # boundary are kept by the rank whose range contains their position)
        ids = [i for i in range(self.R_global) if off[i] < hi and off[i + 1] > lo or (off[i] == off[i + 1] and lo <= off[i] < hi)]
        self.r_lo = ids[0] if ids else 0
        self.r_hi = ids[-1] + 1 if ids else 0
        self.R = self.r_hi - self.r_lo
        loc = np.clip(off[self.r_lo:self.r_hi + 1] - lo, 0, T) if self.R else np.zeros(1, np.int64)
        self.offsets = torch.from_numpy(loc.astype(np.int32)).to(device)
        self.chunk = dz_chunk_rows
        self.shape = make_shape(T, H, V, 0, V, inv_temperature)
        self.params = make_params(max(1, self.R), loss_denominator, alpha, beta, guard, variant, kl_tau, kl_set)
        f32 = dict(dtype=torch.float32, device=device)
        self.logprob, self.entropy, self.lse, self.coef = (torch.empty(T, **f32) for _ in range(4))
        self.keep = torch.empty(T, dtype=torch.uint8, device=device)
        self.guarded = torch.empty(max(1, self.R), dtype=torch.uint8, device=device)
        self.adv_global = torch.empty(self.R_global, **f32)
        self.kmin = torch.empty(max(1, self.R), **f32)
        self.lr = torch.empty(max(1, self.R), dtype=torch.float64, device=device)
        self.n = torch.empty(max(1, self.R), dtype=torch.int32, device=device)
        self.kmin_g = torch.empty(self.R_global, **f32)
        self.lr_g = torch.empty(self.R_global, dtype=torch.float64, device=device)
        self.n_g = torch.empty(self.R_global, dtype=torch.int32, device=device)
        self.report = torch.zeros(48, dtype=torch.uint8, device=device)
        self.d_hidden = torch.empty(T, H, dtype=d_hidden_dtype, device=device)
        self.ws = (alloc_workspace(rl_workspace_bytes(self.shape, max(1, self.R), dz_chunk_rows), device)
                   if workspace else None)
        self.loss_ws = alloc_workspace(48 * max(1, self.R), device) if workspace else None
        self.guarded_global = 0

    def step(self, hidden, w, targets, infer, rewards_global, loss_mask, d_w_vocab):
        """rewards_global: [R_global] rewards of every rollout of the step (group-major).
        Returns d_w_vocab, all-reduced over the group."""
        ph, R, a, b = self.ph, self.R, self.r_lo, self.r_hi
        ph.group_advantages(rewards_global, self.G, self.adv_global)
        ph.logprob_fwd(self.shape, hidden, w, targets, self.logprob, self.entropy, self.lse, workspace=self.ws)
        if R:
            ph.rollout_stats(self.params, self.T, self.V, self.logprob, infer, targets, self.offsets, loss_mask,
                             self.kmin, self.lr, self.n)
        # the rollouts' statistics over every rank that holds part of them
        self.kmin_g.fill_(float("inf"))
        self.lr_g.zero_()
        self.n_g.zero_()
        if R:
            self.kmin_g[a:b] = self.kmin[:R]
            self.lr_g[a:b] = self.lr[:R]
            self.n_g[a:b] = self.n[:R]
        dist.all_reduce(self.kmin_g, op=dist.ReduceOp.MIN, group=self.group)
        dist.all_reduce(self.lr_g, group=self.group)
        dist.all_reduce(self.n_g, group=self.group)
        self.guarded_global = int((self.kmin_g < self.params.guard_threshold).sum().item())
        if R:
            self.kmin[:R] = self.kmin_g[a:b]
            self.lr[:R] = self.lr_g[a:b]
            self.n[:R] = self.n_g[a:b]
            ph.loss_coef_ex(self.params, self.T, self.V, self.logprob, infer, targets, self.adv_global[a:b].contiguous(),
                            self.offsets, loss_mask, self.kmin, self.lr, self.n, self.coef, self.keep, self.guarded,
                            self.report, workspace=self.loss_ws)
        else:
            self.coef.zero_()
            self.keep.zero_()
        ph.bwd_phases(self.shape, hidden, w, targets, self.lse, self.coef, self.d_hidden, d_w_vocab, RL_BWD_ALL,
                      workspace=self.ws)
        dist.all_reduce(d_w_vocab, group=self.group)                                      # the exchange
        return d_w_vocab


def newton_schulz_row_sharded(phases, g_shard, steps=5, group=None, workspace=None, out=None):
    """Muon's Newton-Schulz on a tall matrix whose rows are sharded across `group`
    (e.g. d_w_vocab after the NVLS reduce-scatter): X^T X is the sum of
    the ranks' X_r^T X_r, so per iteration the ranks all-reduce one N x N fp32 Gram
    (and once the sum of squares for ||G||_F) and each updates its own rows. Returns
    this rank's rows of NS(G) in bf16; with one rank it equals rl_newton_schulz."""
    M, N = g_shard.shape
    dev = g_shard.device
    if workspace is None and dev.type == "cuda":
        from . import load_library
        workspace = alloc_workspace(load_library().rl_newton_schulz_workspace_bytes(M, N), dev)
    sumsq = torch.zeros(1, dtype=torch.float64, device=dev)
    gram = torch.empty(N, N, dtype=torch.float32 if dev.type == "cuda" else torch.float64, device=dev)
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16 if dev.type == "cuda" else torch.float64, device=dev)
    phases.ns_sumsq(g_shard, sumsq, workspace)
    dist.all_reduce(sumsq, group=group)                                   # ||G||_F^2
    for j in range(steps):
        phases.ns_gram(j, g_shard, sumsq, gram, workspace)
        dist.all_reduce(gram, group=group)                                # the N x N Gram
        phases.ns_apply(j, steps, gram, M, N, out, workspace)
    return out
