"""The seeded input generator (no method arithmetic): sizes and packing invariants."""
import numpy as np

import synth


def test_rollout_lengths_sum_to_T_even_with_fewer_tokens_than_rollouts():
    for ragged in (False, True):
        wl = synth.Workload("w", 4, 4, 8, 64, 64, ragged=ragged)
        for T in (0, 1, 3, 15, 16, 17, 128, 1000):
            L = synth.rollout_lengths(wl, 3, T)
            assert L.sum() == T and len(L) == wl.num_rollouts and (L >= 0).all()
            if T >= wl.num_rollouts:
                assert (L >= 1).all()


def test_batch_is_reproducible():
    wl = synth.CONFIGS["tiny"]
    a, b = synth.make_batch(wl, 5), synth.make_batch(wl, 5)
    for k in ("hidden", "w_vocab", "targets", "rewards", "rollout_offsets", "loss_mask", "delta_noise", "spikes"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
