"""Rollouts split across ranks (sequence-sharded packed rows) on 2-4 GPUs
against the fp64 oracle of the whole batch (`-m gpu`; skipped with fewer than 2 GPUs).

The packed rows are cut at arbitrary positions, one cut inside a guarded rollout, so
the guard and GSPO's sequence ratio (R17) of a split rollout need the
rollout statistics of every rank that holds part of it: rl_rollout_stats on each rank,
all-reduce (MIN of the min ratio, SUM of log-ratio sums and counts), rl_loss_coef_ex
(parallel.SplitRolloutPolicyLoss). The reassembled logprob / keep / coef / guard flags /
counters / loss / dH / dW are held to harness.compare.
"""
import os
import socket

import numpy as np
import pytest
import torch

import harness
import synth

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs 2 GPUs", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = min(4, torch.cuda.device_count())
WL = synth.Workload("split", 4, 4, 90, 384, 3000, ragged=True, delta_sigma=0.6, spike_rate=4e-3)
VARIANTS = [("icepop", 0.5, 5.0), ("gspo", 0.9, 1.1), ("cispo", 0.8, 1.25)]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    return harness.make_case(WL, 51, targets="sampled", plants=True)


def _bounds(c):
    b = c.batch
    g = harness.run_oracle(c).report.guarded
    gi = int(np.nonzero(g)[0][0])
    cut = int((b.rollout_offsets[gi] + b.rollout_offsets[gi + 1]) // 2)
    rng = np.random.default_rng(5)
    others = rng.choice(np.setdiff1d(np.arange(1, b.T), [cut]), size=WORLD - 2, replace=False).tolist()
    return [0] + sorted([cut] + others) + [b.T], gi


def _worker(rank, port, d):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=dev)
    import paper_2512_16144_b200 as rl
    from paper_2512_16144_b200 import parallel
    z = np.load(os.path.join(d, "case.npz"))
    bounds = z["bounds"]
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).to(dev)  # noqa: E731
    res = {}
    for variant, a, b_ in VARIANTS:
        D = float(len(z["rewards"].reshape(-1))) if variant == "gspo" else float(z["loss_mask"].sum())
        eng = parallel.SplitRolloutPolicyLoss(parallel.LibrlPhases(), T=hi - lo, H=WL.hidden, V=WL.vocab,
                                              global_offsets=z["offsets"], row_start=lo, group_size=WL.group_size,
                                              loss_denominator=D, alpha=a, beta=b_, variant=variant, device=dev)
        dw = torch.empty(WL.vocab, WL.hidden, device=dev)
        eng.step(bf(z["hidden"][lo:hi]), bf(z["w"]), torch.from_numpy(z["targets"][lo:hi].copy()).to(dev),
                 torch.from_numpy(z["infer"][lo:hi].copy()).to(dev),
                 torch.from_numpy(z["rewards"].reshape(-1).copy()).to(dev),
                 torch.from_numpy(z["loss_mask"][lo:hi].copy()).to(dev), dw)
        torch.cuda.synchronize()
        rep = rl.read_report(eng.report).as_dict()
        res[variant] = dict(logprob=eng.logprob.cpu().numpy(), entropy=eng.entropy.cpu().numpy(),
                            lse=eng.lse.cpu().numpy(), coef=eng.coef.cpu().numpy(), keep=eng.keep.cpu().numpy(),
                            guarded=eng.guarded[:eng.R].cpu().numpy(), r_lo=eng.r_lo,
                            dh=eng.d_hidden.float().cpu().numpy(), dw=dw.cpu().numpy(),
                            rep=np.array([rep[k] for k in sorted(rep)]), rep_keys=np.array(sorted(rep)),
                            guarded_global=eng.guarded_global)
        dist.barrier()
    np.savez(os.path.join(d, f"r{rank}.npz"), **{f"{v}__{k}": x for v, r in res.items() for k, x in r.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def split_results(tmp_path_factory):
    d = tmp_path_factory.mktemp("split")
    c = _case()
    bounds, gi = _bounds(c)
    b = c.batch
    np.savez(d / "case.npz", hidden=b.hidden, w=b.w_vocab, targets=b.targets, infer=c.infer, rewards=b.rewards,
             offsets=b.rollout_offsets, loss_mask=b.loss_mask, bounds=np.array(bounds))
    mp.start_processes(_worker, args=(_port(), str(d)), nprocs=WORLD, start_method="spawn")
    return c, d, bounds, gi


@pytest.mark.parametrize("variant,alpha,beta", VARIANTS)
def test_split_rollouts_vs_oracle(split_results, variant, alpha, beta):
    c, d, bounds, gi = split_results
    c.variant, c.alpha, c.beta = variant, alpha, beta
    b = c.batch
    D = float(len(c.adv)) if variant == "gspo" else b.loss_denominator
    ref = harness.run_oracle(c, loss_denominator=D)
    ranks = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(WORLD)]
    get = lambda z, k: z[f"{variant}__{k}"]  # noqa: E731
    gpu = {k: np.concatenate([get(z, k) for z in ranks]) for k in ("logprob", "entropy", "lse", "coef", "keep")}
    gpu["d_hidden"] = np.concatenate([get(z, "dh") for z in ranks]).astype(np.float64)
    for z in ranks[1:]:
        assert np.array_equal(get(z, "dw"), get(ranks[0], "dw"))      # one all-reduced dW
    gpu["d_w_vocab"] = get(ranks[0], "dw").astype(np.float64)
    # the guard flag of every rollout, from whichever rank holds (part of) it: split rollouts agree
    R = len(c.adv)
    guarded = np.full(R, -1)
    for z in ranks:
        r0, gz = int(get(z, "r_lo")), get(z, "guarded")
        for j, v in enumerate(gz):
            assert guarded[r0 + j] in (-1, int(v)), "ranks disagree on a split rollout's guard"
            guarded[r0 + j] = int(v)
    gpu["guarded"] = np.maximum(guarded, 0).astype(np.uint8)
    keys = get(ranks[0], "rep_keys")
    rep = {str(k): sum(float(get(z, "rep")[i]) for z in ranks) for i, k in enumerate(keys)}
    rep["guarded_rollouts"] = int(get(ranks[0], "guarded_global"))     # the exact count (split rollouts once)
    gpu["report"] = {k: (v if k in ("loss", "mismatch_kl_sum") else int(round(v))) for k, v in rep.items()}
    assert ref.report.guarded[gi]                                     # the cut goes through a guarded rollout
    err = harness.compare(c, ref, gpu)
    print("split", variant, WORLD, "bounds", bounds, err)
