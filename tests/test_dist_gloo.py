"""Multi-process (world size 2, 4 and 8, gloo, CPU) checks of the N > 1 host logic in
paper_2512_16144_b200/parallel.py: vocab sharding, rank-ordered partial gather
and merge, redundant S3, dH partial reduction, DP with a global denominator, the
dW reduction, and gradient accumulation over micro-batches with one deferred
reduction. The arithmetic is supplied by `OraclePhases`, a test double
built from the fp64 oracle, so the composition is checked on any machine; the
GPU path runs the same classes with librl's phases (bench.py, N > 1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import oracle.muon
import synth
from paper_2512_16144_b200 import parallel

WORLD = 2
WORLDS = [2, 4, 8]     # 8: the largest NVLS group (RL_NVLS_MAX_RANKS), the driver's 8-GPU scaling run


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OraclePhases:
    """librl's split-phase signatures implemented with oracle functions (CPU)."""

    def group_advantages(self, rewards, G, adv):
        adv.copy_(torch.from_numpy(oracle.group_advantages(rewards.double().numpy().reshape(-1, G)).reshape(-1)))

    def fwd_partials(self, shape, hidden, w_shard, targets, partials, workspace=None):
        Z = oracle.lm_logits(hidden.double().numpy(), w_shard.double().numpy(), shape.inv_temperature)
        m, s, u, zt = oracle.shard_stats(Z, targets.long().numpy(), shape.vocab_offset)
        partials.copy_(torch.from_numpy(np.stack([m, s, u, zt], axis=1)))

    def merge_partials(self, parts, n_parts, T, logprob, entropy, lse):
        p = parts.double().numpy()
        l, e, zt = oracle.merge_shard_stats([tuple(p[j, :, c] for c in range(4)) for j in range(n_parts)])
        logprob.copy_(torch.from_numpy(zt - l))
        entropy.copy_(torch.from_numpy(e))
        lse.copy_(torch.from_numpy(l))

    def loss_coef(self, params, T, V_global, logprob, infer, targets, adv, offsets, loss_mask, coef, keep, guarded,
                  report, workspace=None):
        variant = {v: k for k, v in oracle.LOSS_VARIANTS.items()}[params.variant]
        kl_set = {v: k for k, v in oracle.KL_SETS.items()}[params.kl_set]
        lp, inf = logprob.double().numpy(), infer.double().numpy()
        rep = oracle.variant_loss(variant, lp, inf, adv.double().numpy(), offsets.numpy(), loss_mask.numpy(),
                                  params.alpha, params.beta, params.guard_threshold, params.loss_denominator,
                                  targets=targets.long().numpy(), vocab=V_global)
        rep = oracle.add_kl_term(rep, lp, inf, params.kl_tau, kl_set, params.loss_denominator)
        coef.copy_(torch.from_numpy(rep.coef))
        keep.copy_(torch.from_numpy(rep.keep.astype(np.uint8)))
        guarded.copy_(torch.from_numpy(rep.guarded.astype(np.uint8)))
        self.loss = rep.loss

    def bwd(self, shape, hidden, w_shard, targets, lse, coef, d_hidden_f32, d_w_vocab, dz_chunk_rows=0,
            workspace=None):
        h, W = hidden.double().numpy(), w_shard.double().numpy()
        invT = shape.inv_temperature
        Z = oracle.lm_logits(h, W, invT)
        P = np.exp(Z - lse.double().numpy()[:, None])
        local = targets.long().numpy() - shape.vocab_offset
        inside = (local >= 0) & (local < W.shape[0])
        P[np.nonzero(inside)[0], local[inside]] -= 1.0
        dU = (coef.double().numpy() * invT)[:, None] * P
        d_hidden_f32.copy_(torch.from_numpy(dU @ W))
        d_w_vocab.copy_(torch.from_numpy(dU.T @ h))

    def full_step(self, shape, params, hidden, w, targets, infer, adv, offsets, loss_mask, *, report, logprob,
                  entropy=None, lse=None, coef=None, keep=None, guarded=None, d_hidden=None, d_w_vocab=None,
                  workspace=None, accumulate_dw=False, dz_chunk_rows=0):
        res = oracle.policy_loss_fwd_bwd(hidden.double().numpy(), w.double().numpy(), targets.long().numpy(),
                                         infer.double().numpy(), None, offsets.numpy(), loss_mask.numpy(),
                                         alpha=params.alpha, beta=params.beta,
                                         guard_threshold=params.guard_threshold,
                                         loss_denominator=params.loss_denominator,
                                         inv_temperature=shape.inv_temperature, rollout_adv=adv.double().numpy(),
                                         variant={v: k for k, v in oracle.LOSS_VARIANTS.items()}[params.variant],
                                         kl_tau=params.kl_tau,
                                         kl_set={v: k for k, v in oracle.KL_SETS.items()}[params.kl_set])
        logprob.copy_(torch.from_numpy(res.logp))
        d_hidden.copy_(torch.from_numpy(res.d_hidden))
        if accumulate_dw:
            d_w_vocab.add_(torch.from_numpy(res.d_w_vocab))
        else:
            d_w_vocab.copy_(torch.from_numpy(res.d_w_vocab))
        self.loss = res.report.loss


    # split rollouts (SplitRolloutPolicyLoss); IcePop only in this double
    def logprob_fwd(self, shape, hidden, w, targets, logprob, entropy, lse, workspace=None):
        Z = oracle.lm_logits(hidden.double().numpy(), w.double().numpy(), shape.inv_temperature)
        lp, ent, l = oracle.log_softmax_stats(Z, targets.long().numpy())
        logprob.copy_(torch.from_numpy(lp))
        entropy.copy_(torch.from_numpy(ent))
        lse.copy_(torch.from_numpy(l))

    @staticmethod
    def _valid(V, infer, targets, loss_mask):
        inf, y = infer.double().numpy(), targets.long().numpy()
        return loss_mask.numpy().astype(bool) & np.isfinite(inf) & (inf <= 0) & (y >= 0) & (y < V)

    def rollout_stats(self, params, T, V, logprob, infer, targets, offsets, loss_mask, kmin, logratio_sum, n_valid):
        d = logprob.double().numpy() - infer.double().numpy()
        v = self._valid(V, infer, targets, loss_mask)
        off = offsets.numpy()
        for i in range(len(off) - 1):
            sel = v[off[i]:off[i + 1]]
            di = d[off[i]:off[i + 1]][sel]
            kmin[i] = float(np.exp(di).min()) if di.size else float("inf")
            logratio_sum[i] = float(di.sum())
            n_valid[i] = int(sel.sum())

    def loss_coef_ex(self, params, T, V, logprob, infer, targets, adv, offsets, loss_mask, kmin, logratio_sum,
                     n_valid, coef, keep, guarded, report, workspace=None):
        assert params.variant == 0, "the double implements IcePop only"
        v = self._valid(V, infer, targets, loss_mask)
        k = np.exp(logprob.double().numpy() - infer.double().numpy())
        g = kmin.double().numpy()[: len(offsets) - 1] < params.guard_threshold       # the reduced guard
        rollout_of = np.repeat(np.arange(len(offsets) - 1), np.diff(offsets.numpy()))
        kp = v & (oracle.masking_function(k, params.alpha, params.beta) > 0) & ~g[rollout_of]
        c = np.where(kp, k * adv.double().numpy()[rollout_of] / params.loss_denominator, 0.0)
        coef.copy_(torch.from_numpy(c))
        keep.copy_(torch.from_numpy(kp.astype(np.uint8)))
        guarded[: len(g)] = torch.from_numpy(g.astype(np.uint8))
        self.loss = -float(c.sum())

    def bwd_phases(self, shape, hidden, w, targets, lse, coef, d_hidden, d_w_vocab, phases, max_sms=0,
                   workspace=None):
        self.bwd(shape, hidden, w, targets, lse, coef, d_hidden, d_w_vocab)

    # row-sharded Newton-Schulz (fp64, the oracle's quintic)
    def ns_sumsq(self, g, sumsq, workspace):
        sumsq.fill_(float((g.double() ** 2).sum()))

    def ns_gram(self, j, g, sumsq, gram, workspace):
        if j == 0:
            self.X = g.double().numpy() / (np.sqrt(float(sumsq[0])) + oracle.muon.NS_EPS)
        gram.copy_(torch.from_numpy(self.X.T @ self.X))

    def ns_apply(self, j, steps, gram, M_local, N, out, workspace):
        a, b, c = oracle.muon.NS_COEFFS
        A = gram.double().numpy()
        self.X = self.X @ (a * np.eye(N) + b * A + c * (A @ A))
        if j == steps - 1:
            out.copy_(torch.from_numpy(self.X))


# 4 prompt groups, so 4 DP ranks each hold a whole group; V = 96 splits over 2 or 4 ranks
# 8 prompt groups (whole groups per DP rank at world 2, 4, 8); V = 96 splits into 8 shards
WL = synth.Workload("dist", 8, 4, 12, 32, 96, ragged=True, prompt_frac=0.2, delta_sigma=0.8, spike_rate=0.02)


def _batch():
    b = synth.make_batch(WL, 11)
    h64, w64 = oracle.bf16_to_f64(b.hidden), oracle.bf16_to_f64(b.w_vocab)
    lp, _, _ = oracle.log_softmax_stats(oracle.lm_logits(h64, w64), b.targets)
    infer = synth.compose_infer_logprobs(lp, b.delta_noise, b.spikes)
    return b, h64, w64, infer


def _bf16(bits):
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16)


LOSS_KW = [{}, {"variant": "cispo", "kl_tau": 0.375, "kl_set": "all"}]   # 0.375: exact in the fp32 ABI field


def _vocab_worker(rank, port, out_dir, kw_i=0, world=WORLD):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, h64, w64, infer = _batch()
    vp = parallel.VocabParallelPolicyLoss(OraclePhases(), T=b.T, H=b.H, V_global=b.V, num_rollouts=len(b.rewards.reshape(-1)),
                                          group_size=WL.group_size, loss_denominator=b.loss_denominator,
                                          device="cpu", workspace=False, **LOSS_KW[kw_i])
    lo, hi = vp.vocab_offset, vp.vocab_offset + vp.V_local
    dw = torch.empty(vp.V_local, b.H, dtype=torch.float64)
    for name in ("parts", "d_hidden", "logprob", "entropy", "lse", "coef", "adv"):
        setattr(vp, name, getattr(vp, name).double())
    dh = vp.step(_bf16(b.hidden), _bf16(b.w_vocab[lo:hi]), torch.from_numpy(b.targets), torch.from_numpy(infer),
                 torch.from_numpy(b.rewards.reshape(-1)), torch.from_numpy(b.rollout_offsets),
                 torch.from_numpy(b.loss_mask), dw)
    np.savez(os.path.join(out_dir, f"vp{rank}.npz"), dh=dh.numpy(), dw=dw.numpy(), logprob=vp.logprob.numpy(),
             coef=vp.coef.numpy(), lo=lo, hi=hi)
    dist.destroy_process_group()


def _dp_worker(rank, port, out_dir, kw_i=0, world=WORLD):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, h64, w64, infer = _batch()
    # rank r takes WL.num_prompts / world whole prompt groups (the guard stays local)
    G = WL.group_size
    per = WL.num_prompts // world
    r0, r1 = rank * per * G, (rank + 1) * per * G
    t0, t1 = int(b.rollout_offsets[r0]), int(b.rollout_offsets[r1])
    lm = torch.from_numpy(b.loss_mask[t0:t1].copy())
    D = parallel.DataParallelPolicyLoss.global_denominator(lm)
    dp = parallel.DataParallelPolicyLoss(OraclePhases(), T=t1 - t0, H=b.H, V=b.V, num_rollouts=r1 - r0, group_size=G,
                                         loss_denominator=D, device="cpu", d_hidden_dtype=torch.float64,
                                         workspace=False, **LOSS_KW[kw_i])
    for name in ("logprob", "entropy", "lse", "coef", "adv"):
        setattr(dp, name, getattr(dp, name).double())
    dw = torch.empty(b.V, b.H, dtype=torch.float64)
    offs = torch.from_numpy((b.rollout_offsets[r0:r1 + 1] - t0).astype(np.int32))
    dp.step(_bf16(b.hidden[t0:t1]), _bf16(b.w_vocab), torch.from_numpy(b.targets[t0:t1].copy()),
            torch.from_numpy(infer[t0:t1].copy()), torch.from_numpy(b.rewards[rank * per:(rank + 1) * per].reshape(-1).copy()),
            offs, lm, dw)
    loss = torch.tensor([dp.ph.loss], dtype=torch.float64)
    dist.all_reduce(loss)
    np.savez(os.path.join(out_dir, f"dp{rank}.npz"), dh=dp.d_hidden.numpy(), dw=dw.numpy(), t0=t0, t1=t1,
             loss=loss.numpy(), D=D)
    dist.destroy_process_group()


def _reference(kw_i=0):
    b, h64, w64, infer = _batch()
    return b, oracle.policy_loss_fwd_bwd(h64, w64, b.targets, infer.astype(np.float64), b.rewards,
                                         b.rollout_offsets, b.loss_mask, **LOSS_KW[kw_i])


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("kw_i", range(len(LOSS_KW)))
def test_vocab_parallel_composition(tmp_path, kw_i, world):
    if world == 8 and kw_i:
        pytest.skip("world 8 runs the paper's loss only (keeps the CPU suite short)")
    mp.start_processes(_vocab_worker, args=(_free_port(), str(tmp_path), kw_i, world), nprocs=world,
                       start_method="spawn")
    b, ref = _reference(kw_i)
    outs = [np.load(tmp_path / f"vp{r}.npz") for r in range(world)]
    for o in outs:   # S2/S3 are identical on every rank; dH is the reduced sum
        np.testing.assert_allclose(o["logprob"], ref.logp, atol=1e-6)
        np.testing.assert_allclose(o["coef"], ref.report.coef, atol=1e-9)
        np.testing.assert_allclose(o["dh"], ref.d_hidden, atol=1e-9)
    dw = np.concatenate([o["dw"] for o in outs])
    np.testing.assert_allclose(dw, ref.d_w_vocab, atol=1e-9)
    assert [int(o["lo"]) for o in outs] == [r * (b.V // world) for r in range(world)]


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("kw_i", range(len(LOSS_KW)))
def test_data_parallel_composition(tmp_path, kw_i, world):
    if world == 8 and kw_i:
        pytest.skip("world 8 runs the paper's loss only (keeps the CPU suite short)")
    mp.start_processes(_dp_worker, args=(_free_port(), str(tmp_path), kw_i, world), nprocs=world,
                       start_method="spawn")
    b, ref = _reference(kw_i)
    outs = [np.load(tmp_path / f"dp{r}.npz") for r in range(world)]
    for o in outs:
        assert float(o["D"]) == b.loss_denominator            # global D, reading R5
        np.testing.assert_allclose(o["dw"], ref.d_w_vocab, atol=1e-12)   # all-reduced dW
        np.testing.assert_allclose(o["dh"], ref.d_hidden[int(o["t0"]):int(o["t1"])], atol=1e-12)
        assert float(o["loss"][0]) == pytest.approx(ref.report.loss, abs=1e-12)


def _dp_micro_worker(rank, port, out_dir):
    """Rank r holds prompt groups 2r and 2r+1 and runs them as two micro-batches
    (one engine per micro-batch shape): dW accumulates locally (accumulate=True on
    the second) and is reduced once, on the last (reduce=False on the first)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    b, h64, w64, infer = _batch()
    G = WL.group_size
    per = WL.num_prompts // WORLD
    off = b.rollout_offsets
    mine = off[rank * per * G], off[(rank + 1) * per * G]
    D = parallel.DataParallelPolicyLoss.global_denominator(torch.from_numpy(b.loss_mask[mine[0]:mine[1]].copy()))
    dw = torch.full((b.V, b.H), float("nan"), dtype=torch.float64)   # overwritten by the first micro-batch
    dh, losses = [], 0.0
    for j in range(per):
        g = rank * per + j
        t0, t1 = int(off[g * G]), int(off[(g + 1) * G])
        dp = parallel.DataParallelPolicyLoss(OraclePhases(), T=t1 - t0, H=b.H, V=b.V, num_rollouts=G, group_size=G,
                                             loss_denominator=D, device="cpu", d_hidden_dtype=torch.float64,
                                             workspace=False)
        for name in ("logprob", "entropy", "lse", "coef", "adv"):
            setattr(dp, name, getattr(dp, name).double())
        offs = torch.from_numpy((off[g * G:(g + 1) * G + 1] - t0).astype(np.int32))
        dp.step(_bf16(b.hidden[t0:t1]), _bf16(b.w_vocab), torch.from_numpy(b.targets[t0:t1].copy()),
                torch.from_numpy(infer[t0:t1].copy()), torch.from_numpy(b.rewards[g].copy()), offs,
                torch.from_numpy(b.loss_mask[t0:t1].copy()), dw, accumulate=j > 0, reduce=j == per - 1)
        if j < per - 1:   # nothing reduced yet: the buffer holds this rank's own partial sum
            assert np.isfinite(dw.numpy()).all()
        dh.append(dp.d_hidden.numpy().copy())
        losses += dp.ph.loss
    loss = torch.tensor([losses], dtype=torch.float64)
    dist.all_reduce(loss)
    np.savez(os.path.join(out_dir, f"mb{rank}.npz"), dh=np.concatenate(dh), dw=dw.numpy(), t0=mine[0], t1=mine[1],
             loss=loss.numpy())
    dist.destroy_process_group()


def test_data_parallel_microbatch_accumulation(tmp_path):
    """Two micro-batches per rank with the reduction deferred to the last equal the
    oracle's gradient of the whole batch (the gradient is linear in the rows, and D
    is the global loss-token count of the step, reading R5)."""
    mp.start_processes(_dp_micro_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, start_method="spawn")
    b, ref = _reference(0)
    for r in range(WORLD):
        o = np.load(tmp_path / f"mb{r}.npz")
        np.testing.assert_allclose(o["dw"], ref.d_w_vocab, atol=1e-12)
        np.testing.assert_allclose(o["dh"], ref.d_hidden[int(o["t0"]):int(o["t1"])], atol=1e-12)
        assert float(o["loss"][0]) == pytest.approx(ref.report.loss, abs=1e-12)


def _ns_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    G = np.random.default_rng(3).standard_normal((96, 16))
    rows = np.array_split(np.arange(96), WORLD)[rank]
    out = parallel.newton_schulz_row_sharded(OraclePhases(), torch.from_numpy(G[rows].copy()), steps=5)
    np.save(os.path.join(out_dir, f"ns{rank}.npy"), out.numpy())
    dist.destroy_process_group()


def test_row_sharded_newton_schulz_composition(tmp_path):
    """Sharding rows and all-reducing the Gram (and ||G||^2) is Newton-Schulz of the
    full matrix: X^T X = sum_r X_r^T X_r (oracle.newton_schulz, fp64)."""
    mp.start_processes(_ns_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"ns{r}.npy") for r in range(WORLD)])
    G = np.random.default_rng(3).standard_normal((96, 16))
    np.testing.assert_allclose(got, oracle.muon.newton_schulz(G, 5), rtol=0, atol=1e-12)


# ---------------------------------------------- rollouts split across ranks (§8(e))
def _split_worker(rank, port, out_dir, bounds):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    world = len(bounds) - 1
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, h64, w64, infer = _batch()
    lo, hi = bounds[rank], bounds[rank + 1]
    eng = parallel.SplitRolloutPolicyLoss(OraclePhases(), T=hi - lo, H=b.H, V=b.V, global_offsets=b.rollout_offsets,
                                          row_start=lo, group_size=WL.group_size,
                                          loss_denominator=b.loss_denominator, device="cpu",
                                          d_hidden_dtype=torch.float64, workspace=False)
    for name in ("logprob", "entropy", "lse", "coef", "adv_global", "kmin", "kmin_g"):
        setattr(eng, name, getattr(eng, name).double())
    dw = torch.empty(b.V, b.H, dtype=torch.float64)
    eng.step(_bf16(b.hidden[lo:hi]), _bf16(b.w_vocab), torch.from_numpy(b.targets[lo:hi].copy()),
             torch.from_numpy(infer[lo:hi].copy()), torch.from_numpy(b.rewards.reshape(-1).copy()),
             torch.from_numpy(b.loss_mask[lo:hi].copy()), dw)
    loss = torch.tensor([getattr(eng.ph, "loss", 0.0)], dtype=torch.float64)
    dist.all_reduce(loss)
    np.savez(os.path.join(out_dir, f"sp{rank}.npz"), dh=eng.d_hidden.numpy(), dw=dw.numpy(), coef=eng.coef.numpy(),
             loss=loss.numpy(), guarded=eng.guarded_global, R=eng.R)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_split_rollout_composition(tmp_path, world):
    """Packed rows split at arbitrary positions, cutting through rollouts (one boundary
    inside a guarded rollout): the ranks' coefficients, dH rows, all-reduced dW and the
    summed loss equal the oracle of the whole batch, and the guard decision of a split
    rollout is the whole rollout's (the reduced min ratio)."""
    b, ref = _reference(0)
    T = b.T
    g = np.nonzero(ref.report.guarded)[0]
    assert len(g), "the batch needs a guarded rollout"
    gi = int(g[len(g) // 2])
    cut = int((b.rollout_offsets[gi] + b.rollout_offsets[gi + 1]) // 2)        # inside a guarded rollout
    assert b.rollout_offsets[gi] < cut < b.rollout_offsets[gi + 1]
    rng = np.random.default_rng(world)
    others = sorted(rng.choice(np.setdiff1d(np.arange(1, T), [cut]), size=world - 2, replace=False).tolist())
    bounds = [0] + sorted([cut] + others) + [T]
    mp.start_processes(_split_worker, args=(_free_port(), str(tmp_path), bounds), nprocs=world, start_method="spawn")
    outs = [np.load(tmp_path / f"sp{r}.npz") for r in range(world)]
    np.testing.assert_allclose(np.concatenate([o["coef"] for o in outs]), ref.report.coef, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([o["dh"] for o in outs]), ref.d_hidden, atol=1e-12)
    for o in outs:
        np.testing.assert_allclose(o["dw"], ref.d_w_vocab, atol=1e-12)
        assert float(o["loss"][0]) == pytest.approx(ref.report.loss, abs=1e-12)
        assert int(o["guarded"]) == int(ref.report.guarded_rollouts)

