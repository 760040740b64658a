"""Multi-GPU composition of the step: one process per GPU,
torch.distributed process groups (NCCL over NVLink) for the collectives, librl's
split-phase C calls for all arithmetic.

* DataParallelPolicyLoss — each rank runs the whole step on its own rollouts
  (whole groups per rank, so the guard and the advantages stay local) with the
  GLOBAL loss denominator D (reading R5); the exchange step is the dW all-reduce.
* VocabParallelPolicyLoss — W row-sharded; K1 partials (16 B/token) are
  all-gathered and merged in rank order; S3 runs redundantly; the dH partials
  are all-reduced; each rank keeps its complete dW shard.

The arithmetic goes through a `phases` object with librl's split-phase
signatures. `LibrlPhases` (the C ABI) is the only implementation in the
package; tests substitute a CPU double to check this host logic on gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (make_params, make_shape, rl_bwd, rl_fwd_partials, rl_group_advantages, rl_last_launch_count,
               rl_loss_coef, rl_merge_partials, rl_policy_loss_fwd_bwd, rl_workspace_bytes, alloc_workspace)


class LibrlPhases:
    """The split phases backed by librl (device tensors, current stream)."""

    def __init__(self):
        self.launches = 0

    def _count(self):
        self.launches += rl_last_launch_count()

    def group_advantages(self, rewards, group_size, adv):
        rl_group_advantages(rewards, group_size, adv)
        self._count()

    def fwd_partials(self, shape, hidden, w_shard, targets, partials, workspace=None):
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

    def bwd(self, shape, hidden, w_shard, targets, lse, coef, d_hidden_f32, d_w_vocab, dz_chunk_rows=0,
            workspace=None):
        rl_bwd(shape, hidden, w_shard, targets, lse, coef, d_hidden_f32=d_hidden_f32, d_w_vocab=d_w_vocab,
               dz_chunk_rows=dz_chunk_rows, workspace=workspace)
        self._count()

    def full_step(self, shape, params, hidden, w, targets, infer, adv, offsets, loss_mask, *, report, logprob,
                  entropy=None, lse=None, coef=None, keep=None, guarded=None, d_hidden=None, d_w_vocab=None,
                  workspace=None):
        rl_policy_loss_fwd_bwd(shape, params, hidden, w, targets, infer, adv, offsets, loss_mask, report=report,
                               logprob=logprob, entropy=entropy, lse=lse, coef=coef, token_keep=keep,
                               rollout_guarded=guarded, d_hidden=d_hidden, d_w_vocab=d_w_vocab,
                               workspace=workspace)
        self._count()


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
                 workspace=True):
        self.ph = phases
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if V_global % self.world:
            raise ValueError("V_global must divide evenly across the vocab-parallel ranks")
        self.V_local = V_global // self.world
        self.vocab_offset = self.rank * self.V_local
        self.T, self.H, self.V_global, self.R, self.G = T, H, V_global, num_rollouts, group_size
        self.shape = make_shape(T, H, self.V_local, self.vocab_offset, V_global, inv_temperature)
        self.params = make_params(num_rollouts, loss_denominator, alpha, beta, guard)
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
        self.d_hidden = torch.empty(T, H, **f32)
        self.ws = self.loss_ws = None
        if workspace:
            self.ws = alloc_workspace(rl_workspace_bytes(self.shape, num_rollouts, dz_chunk_rows), dev)
            self.loss_ws = alloc_workspace(48 * max(1, num_rollouts), dev)

    def step(self, hidden, w_shard, targets, infer, rewards, offsets, loss_mask, d_w_vocab):
        ph = self.ph
        ph.group_advantages(rewards, self.G, self.adv)
        ph.fwd_partials(self.shape, hidden, w_shard, targets, self.parts[self.rank], workspace=self.ws)
        _all_gather_rows(self.parts, self.parts[self.rank], self.group)                 # exchange 1
        ph.merge_partials(self.parts, self.world, self.T, self.logprob, self.entropy, self.lse)
        ph.loss_coef(self.params, self.T, self.V_global, self.logprob, infer, targets, self.adv, offsets,
                     loss_mask, self.coef, self.keep, self.guarded, self.report, workspace=self.loss_ws)
        ph.bwd(self.shape, hidden, w_shard, targets, self.lse, self.coef, self.d_hidden, d_w_vocab,
               dz_chunk_rows=self.chunk, workspace=self.ws)
        dist.all_reduce(self.d_hidden, group=self.group)                                  # exchange 2
        return self.d_hidden


class DataParallelPolicyLoss:
    """S0..S6 on each rank's own rollouts; dW summed over the ranks of `group`."""

    def __init__(self, phases, *, T, H, V, num_rollouts, group_size, loss_denominator, group=None,
                 inv_temperature=1.0, alpha=0.5, beta=5.0, guard=1e-5, device=None, d_hidden_dtype=torch.bfloat16,
                 workspace=True):
        self.ph = phases
        self.group = group
        self.world = dist.get_world_size(group)
        self.T, self.H, self.V, self.R, self.G = T, H, V, num_rollouts, group_size
        self.shape = make_shape(T, H, V, 0, V, inv_temperature)
        self.params = make_params(num_rollouts, loss_denominator, alpha, beta, guard)
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
        self.ws = alloc_workspace(rl_workspace_bytes(self.shape, num_rollouts), dev) if workspace else None

    @staticmethod
    def global_denominator(loss_mask: torch.Tensor, group=None) -> float:
        """D = sum over ranks of the local loss-token counts (one all-reduce at batch assembly)."""
        t = loss_mask.to(torch.float64).sum().reshape(1)
        dist.all_reduce(t, group=group)
        return float(t.item())

    def step(self, hidden, w, targets, infer, rewards, offsets, loss_mask, d_w_vocab):
        ph = self.ph
        ph.group_advantages(rewards, self.G, self.adv)
        ph.full_step(self.shape, self.params, hidden, w, targets, infer, self.adv, offsets, loss_mask,
                     report=self.report, logprob=self.logprob, entropy=self.entropy, lse=self.lse, coef=self.coef,
                     keep=self.keep, guarded=self.guarded, d_hidden=self.d_hidden, d_w_vocab=d_w_vocab,
                     workspace=self.ws)
        dist.all_reduce(d_w_vocab, group=self.group)                                      # the exchange
        return d_w_vocab
