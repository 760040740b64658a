"""fp64 CPU oracle of PAPER.md §3.3 (Eq.1, Eq.2) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. It shares no code with the CUDA path.
"""
from .icepop import (  # noqa: F401
    KL_SETS, LOSS_VARIANTS, LossReport, StepResult, add_kl_term, cispo_loss, gspo_loss, variant_loss, bf16_to_f64, group_advantages, icepop_backward, icepop_loss,
    lm_logits, log_softmax_stats, masking_function, merge_shard_stats, policy_loss_fwd_bwd,
    rollout_guard, shard_stats, validate_offsets,
)
