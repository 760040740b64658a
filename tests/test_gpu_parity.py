"""CUDA path vs the fp64 oracle, element by element, through the C ABI (`-m gpu`).

Sizes span several 128x256 tiles with ragged tails in T, V and H (K), and the
BASELINE.json tiny config; edge cases: empty batch, empty rollouts, malformed
offsets, non-finite stored log-probs, out-of-range targets, loss-mask rows,
temperature, chunked backward, gradient accumulation, fp32 dH, determinism.
"""
import numpy as np
import pytest

import harness
import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

TINY = synth.CONFIGS["tiny"]
RAGGED = synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8,
                        spike_rate=0.02)


def test_group_advantages_vs_oracle():
    rng = np.random.default_rng(0)
    for Np, G in ((2, 4), (37, 16), (5, 2), (3, 33)):
        S = (rng.random((Np, G)) < 0.5).astype(np.float32)
        S[:, 0] = 0.3  # non-binary values too
        got = rl.rl_group_advantages(torch.from_numpy(S.reshape(-1)).cuda(), G).cpu().numpy()
        ref = oracle.group_advantages(S.astype(np.float64)).reshape(-1)
        np.testing.assert_allclose(got, ref, atol=1e-7)
    with pytest.raises(rl.RLError):
        rl.rl_group_advantages(torch.zeros(4, device="cuda"), 1)


@pytest.mark.parametrize("wl,tokens,vocab,hidden,invT", [
    (TINY, None, None, None, 1.0),
    (RAGGED, 333, 1000, 200, 1.0),
    (RAGGED, 333, 1000, 200, 1 / 0.7),
    (synth.Workload("mid", 2, 8, 80, 512, 4184, ragged=True, delta_sigma=1.0, spike_rate=1e-3), None, None, None, 1.0),
])
def test_logprob_fwd(wl, tokens, vocab, hidden, invT):
    c = harness.make_case(wl, 1, tokens=tokens, vocab=vocab, hidden=hidden, inv_temperature=invT)
    ref = harness.run_oracle(c, backward=False)
    d = harness.to_device(c)
    b = c.batch
    shape = rl.make_shape(b.T, b.H, b.V, 0, b.V, invT)
    lp, ent, lse = (torch.empty(b.T, device="cuda") for _ in range(3))
    rl.rl_logprob_fwd(shape, d["hidden"], d["w"], d["targets"], lp, ent, lse)
    torch.cuda.synchronize()
    assert np.max(np.abs(lp.cpu().numpy() - ref.logp)) <= harness.LOGP_TOL
    assert np.max(np.abs(ent.cpu().numpy() - ref.entropy)) <= harness.LOGP_TOL
    assert np.max(np.abs(lse.cpu().numpy() - ref.lse)) <= harness.LOGP_TOL


@pytest.mark.parametrize("wl,tokens,vocab,hidden,invT", [
    (TINY, None, None, None, 1.0),
    (RAGGED, 333, 1000, 200, 1 / 0.7),
    (RAGGED, 333, 1000, 392, 1.0),            # one partial 256x512 (wide) tile in N for K5/K6
    (RAGGED, 517, 1300, 776, 1.0),            # one full + one partial wide tile
    (synth.Workload("mid", 2, 8, 80, 512, 4184, ragged=True, prompt_frac=0.1, delta_sigma=1.0,
                    spike_rate=1e-3), None, None, None, 1.0),
])
def test_policy_loss_step(wl, tokens, vocab, hidden, invT):
    c = harness.make_case(wl, 2, tokens=tokens, vocab=vocab, hidden=hidden, inv_temperature=invT)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c)
    err = harness.compare(c, ref, gpu)
    print(err)
    assert gpu["launches"] > 0


def test_step_fp32_dh_and_accumulate():
    c = harness.make_case(RAGGED, 3, tokens=300, vocab=1000, hidden=200)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c, dh_f32=True)
    harness.compare(c, ref, gpu)
    init = torch.from_numpy(np.random.default_rng(0).standard_normal((1000, 200)).astype(np.float32)).cuda()
    gpu2 = harness.run_gpu_step(c, dh_f32=True, accumulate_dw=True, dw_init=init)
    got = gpu2["d_w_vocab"] - init.cpu().numpy().astype(np.float64)
    assert harness.rel_fro(got, ref.d_w_vocab) <= 2e-2


def test_chunked_backward_matches():
    c = harness.make_case(RAGGED, 4, tokens=333, vocab=1000, hidden=200)
    ref = harness.run_oracle(c)
    d = harness.to_device(c)
    b = c.batch
    T, H, V = b.T, b.H, b.V
    shape = rl.make_shape(T, H, V, 0, V)
    lse = torch.from_numpy(ref.lse.astype(np.float32)).cuda()
    coef = torch.from_numpy(ref.report.coef.astype(np.float32)).cuda()
    for chunk in (0, 128, 100):
        dh = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        dw = torch.empty(V, H, device="cuda")
        rl.rl_bwd(shape, d["hidden"], d["w"], d["targets"], lse, coef, d_hidden=dh, d_w_vocab=dw,
                  dz_chunk_rows=chunk)
        torch.cuda.synchronize()
        assert harness.rel_fro(dh.float().cpu().numpy(), ref.d_hidden) <= harness.GRAD_RTOL
        assert harness.rel_fro(dw.cpu().numpy(), ref.d_w_vocab) <= harness.GRAD_RTOL
        # invariant: sum_v dW[v, :] = 0 (oracle gives ~1e-16); bf16 dU leaves ~1e-3
        assert np.linalg.norm(dw.cpu().numpy().sum(0)) / np.linalg.norm(dw.cpu().numpy()) < 1e-2


def test_determinism_bitwise():
    c = harness.make_case(RAGGED, 5, tokens=333, vocab=1000, hidden=200)
    g1 = harness.run_gpu_step(c)
    g2 = harness.run_gpu_step(c)
    for k in ("logprob", "entropy", "coef", "keep", "d_hidden", "d_w_vocab"):
        assert np.array_equal(g1[k], g2[k]), k
    assert g1["report"] == g2["report"]


def test_faults_are_counted_and_neutralised():
    def corrupt(b, infer):
        infer[3] = np.nan
        infer[10] = np.inf
        infer[11] = 0.25          # positive stored log-prob
        b.targets[20] = -1
        b.targets[21] = b.V + 5
    c = harness.make_case(RAGGED, 6, tokens=120, vocab=1000, hidden=64, corrupt=corrupt)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c)
    assert gpu["report"]["nonfinite_inputs"] == ref.report.nonfinite_inputs > 0
    assert gpu["report"]["bad_targets"] == ref.report.bad_targets == 2
    ok = np.ones(c.batch.T, bool)
    ok[[20, 21]] = False   # logprob of an out-of-range target is undefined
    assert np.max(np.abs(gpu["logprob"][ok] - ref.logp[ok])) <= harness.LOGP_TOL
    for t in (3, 10, 11, 20, 21):
        assert gpu["coef"][t] == 0.0 and gpu["keep"][t] == 0
    assert abs(gpu["report"]["loss"] - ref.report.loss) <= harness.LOSS_TOL


def test_bad_offsets_neutralise():
    c = harness.make_case(RAGGED, 7, tokens=120, vocab=1000, hidden=64)
    c.batch.rollout_offsets[2], c.batch.rollout_offsets[3] = c.batch.rollout_offsets[3], c.batch.rollout_offsets[2]
    gpu = harness.run_gpu_step(c)
    assert gpu["report"]["bad_offsets"] == 1
    assert not gpu["coef"].any() and gpu["report"]["loss"] == 0.0
    assert not np.any(gpu["d_hidden"]) and not np.any(gpu["d_w_vocab"])


def test_empty_rollouts_and_all_masked_rows():
    def corrupt(b, infer):
        b.rollout_offsets[1:4] = b.rollout_offsets[1]   # rollouts 1, 2 empty
        b.loss_mask[: b.rollout_offsets[1]] = 0          # rollout 0 all prompt
    c = harness.make_case(RAGGED, 8, tokens=200, vocab=1000, hidden=64, corrupt=corrupt)
    ref = harness.run_oracle(c)
    gpu = harness.run_gpu_step(c)
    harness.compare(c, ref, gpu)


def test_empty_batch():
    H, V = 64, 1000
    shape = rl.make_shape(0, H, V, 0, V)
    params = rl.make_params(2, 1.0)
    report = rl.new_report()
    dw = torch.full((V, H), 7.0, device="cuda")
    off = torch.zeros(3, dtype=torch.int32, device="cuda")
    adv = torch.zeros(2, device="cuda")
    w = torch.zeros(V, H, dtype=torch.bfloat16, device="cuda")
    e = torch.empty(0, device="cuda")
    rl.rl_policy_loss_fwd_bwd(shape, params, None, w, None, None, adv, off, None, report=report, logprob=e,
                              d_w_vocab=dw)
    torch.cuda.synchronize()
    r = rl.read_report(report).as_dict()
    assert r["loss"] == 0.0 and r["kept_tokens"] == 0 and r["bad_offsets"] == 0
    assert not dw.any()


def test_uniform_logits_closed_form_on_gpu():
    """W = 0 -> logprob = -ln V and entropy = ln V exactly up to fp32."""
    T, H, V = 300, 64, 1000
    hidden = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    w = torch.zeros(V, H, dtype=torch.bfloat16, device="cuda")
    tg = torch.randint(0, V, (T,), dtype=torch.int32, device="cuda")
    lp, ent = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    rl.rl_logprob_fwd(rl.make_shape(T, H, V), hidden, w, tg, lp, ent)
    torch.cuda.synchronize()
    assert np.allclose(lp.cpu().numpy(), -np.log(V), atol=1e-5)
    assert np.allclose(ent.cpu().numpy(), np.log(V), atol=1e-5)


def test_vocab_parallel_split_phases_single_gpu():
    """Emulate n vocab shards on one GPU through the split-phase ABI; the merge of
    the shards' partials and the sum of dH partials must equal the oracle."""
    c = harness.make_case(RAGGED, 9, tokens=333, vocab=1000, hidden=200)
    ref = harness.run_oracle(c)
    d = harness.to_device(c)
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    cuts = [0, 256, 600, 1000]
    parts = torch.empty(len(cuts) - 1, T, 4, device="cuda")
    for j, (a, e) in enumerate(zip(cuts[:-1], cuts[1:])):
        shp = rl.make_shape(T, H, e - a, a, V)
        rl.rl_fwd_partials(shp, d["hidden"], d["w"][a:e].contiguous(), d["targets"], parts[j])
    lp, ent, lse = (torch.empty(T, device="cuda") for _ in range(3))
    rl.rl_merge_partials(parts, len(cuts) - 1, T, lp, ent, lse)
    coef = torch.empty(T, device="cuda")
    keep = torch.empty(T, dtype=torch.uint8, device="cuda")
    guarded = torch.empty(R, dtype=torch.uint8, device="cuda")
    report = rl.new_report()
    params = rl.make_params(R, b.loss_denominator)
    rl.rl_loss_coef(params, T, V, lp, d["infer"], d["targets"], d["adv"], d["offsets"], d["loss_mask"], coef,
                    keep, guarded, report=report)
    dh = torch.zeros(T, H, device="cuda")
    dws = []
    for a, e in zip(cuts[:-1], cuts[1:]):
        shp = rl.make_shape(T, H, e - a, a, V)
        dhp = torch.empty(T, H, device="cuda")
        dw = torch.empty(e - a, H, device="cuda")
        rl.rl_bwd(shp, d["hidden"], d["w"][a:e].contiguous(), d["targets"], lse, coef, d_hidden_f32=dhp,
                  d_w_vocab=dw)
        dh += dhp
        dws.append(dw)
    torch.cuda.synchronize()
    gpu = dict(logprob=lp.cpu().numpy(), entropy=ent.cpu().numpy(), lse=lse.cpu().numpy(),
               coef=coef.cpu().numpy(), keep=keep.cpu().numpy(), guarded=guarded.cpu().numpy(),
               report=rl.read_report(report).as_dict(), d_hidden=dh.cpu().numpy().astype(np.float64),
               d_w_vocab=torch.cat(dws).cpu().numpy().astype(np.float64))
    harness.compare(c, ref, gpu)


def test_hostio_matches_device_path():
    c = harness.make_case(RAGGED, 10, tokens=333, vocab=1000, hidden=200)
    gdev = harness.run_gpu_step(c)
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    d = harness.to_device(c)
    shape = rl.make_shape(T, H, V)
    params = rl.make_params(R, b.loss_denominator)
    report = rl.new_report()
    dh = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(V, H, device="cuda")
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    rep = rl.rl_policy_loss_fwd_bwd_hostio(
        shape, params, b.wl.group_size, pin(b.hidden.view(np.int16)), d["w"], pin(b.targets), pin(c.infer),
        pin(b.rewards.reshape(-1)), pin(b.rollout_offsets), pin(b.loss_mask), report=report, d_hidden=dh,
        d_w_vocab=dw)
    assert rep.as_dict() == gdev["report"]
    assert np.array_equal(dh.float().cpu().numpy(), gdev["d_hidden"])
    assert np.array_equal(dw.cpu().numpy(), gdev["d_w_vocab"])


def test_host_validation_errors():
    shape = rl.make_shape(10, 60, 100)   # H not a multiple of 8
    with pytest.raises(rl.RLError) as e:
        rl.rl_logprob_fwd(shape, torch.zeros(10, 60, dtype=torch.bfloat16, device="cuda"),
                          torch.zeros(100, 60, dtype=torch.bfloat16, device="cuda"),
                          torch.zeros(10, dtype=torch.int32, device="cuda"), torch.empty(10, device="cuda"))
    assert e.value.status == 2
    shape = rl.make_shape(10, 64, 100)
    with pytest.raises(rl.RLError) as e:
        rl.rl_logprob_fwd(shape, torch.zeros(10, 64, dtype=torch.bfloat16, device="cuda"),
                          torch.zeros(100, 64, dtype=torch.bfloat16, device="cuda"),
                          torch.zeros(10, dtype=torch.int32, device="cuda"), torch.empty(10, device="cuda"),
                          workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))
    assert e.value.status == 5


def test_no_out_of_bounds_writes_guard_bands():
    """compute-sanitizer is unavailable on the GPU pool, so every output (and the
    workspace) sits inside a larger buffer whose margins hold a sentinel; ragged
    T, V, H exercise every tail path. Any byte written outside the tensors fails."""
    c = harness.make_case(RAGGED, 12, tokens=333, vocab=1000, hidden=200)
    d = harness.to_device(c)
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    G = 4096   # guard elements on each side (16 KB of fp32)

    def guarded(n, dtype):
        buf = torch.full((n + 2 * G,), 0, dtype=dtype, device="cuda")
        buf.view(torch.uint8).fill_(0xA5)
        return buf, buf[G:G + n]

    bufs = {}
    f32 = torch.float32
    for name, n, dt in (("logprob", T, f32), ("entropy", T, f32), ("lse", T, f32), ("coef", T, f32),
                        ("keep", T, torch.uint8), ("guarded", R, torch.uint8), ("report", 48, torch.uint8),
                        ("dh", T * H, torch.bfloat16), ("dw", V * H, f32)):
        bufs[name] = guarded(n, dt)
    shape = rl.make_shape(T, H, V)
    params = rl.make_params(R, b.loss_denominator)
    wsn = rl.rl_workspace_bytes(shape, R)
    wbuf, ws = guarded(wsn + (16 - wsn % 16) % 16, torch.uint8)
    v = {k: x[1] for k, x in bufs.items()}
    rl.rl_policy_loss_fwd_bwd(shape, params, d["hidden"], d["w"], d["targets"], d["infer"], d["adv"], d["offsets"],
                              d["loss_mask"], report=v["report"], logprob=v["logprob"], entropy=v["entropy"],
                              lse=v["lse"], coef=v["coef"], token_keep=v["keep"], rollout_guarded=v["guarded"],
                              d_hidden=v["dh"].view(T, H), d_w_vocab=v["dw"].view(V, H), workspace=ws)
    torch.cuda.synchronize()
    for name, (buf, _) in list(bufs.items()) + [("workspace", (wbuf, None))]:
        raw = buf.view(torch.uint8)
        esz = buf.element_size()
        head, tail = raw[: G * esz], raw[raw.numel() - G * esz:]
        assert bool((head == 0xA5).all()) and bool((tail == 0xA5).all()), f"write outside {name}"


@pytest.mark.parametrize("variant,lo,hi", [("cispo", 0.8, 1.25), ("gspo", 0.9, 1.1), ("gspo", 0.5, 2.0)])
def test_loss_variants_vs_oracle(variant, lo, hi):
    """CISPO and GSPO coefficients (S3 only; same backward kernels)."""
    c = harness.make_case(RAGGED, 13, tokens=333, vocab=1000, hidden=200)
    c.variant, c.alpha, c.beta = variant, lo, hi
    D = float(len(c.adv)) if variant == "gspo" else c.batch.loss_denominator
    ref = harness.run_oracle(c, loss_denominator=D)
    gpu = harness.run_gpu_step(c, loss_denominator=D)
    err = harness.compare(c, ref, gpu)
    if hi - lo < 0.5:
        assert ref.report.masked_low + ref.report.masked_high > 0      # the clip is exercised
    print(variant, err)


def test_cuda_graph_capture_replays_the_step():
    """The device-side step is capturable in a CUDA graph (no host syncs, no
    allocations): replay on new inputs equals an eager call bitwise."""
    c = harness.make_case(RAGGED, 14, tokens=333, vocab=1000, hidden=200)
    d = harness.to_device(c)
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    shape = rl.make_shape(T, H, V)
    params = rl.make_params(R, b.loss_denominator)
    ws = rl.alloc_workspace(rl.rl_workspace_bytes(shape, R))
    out = {k: torch.empty(T, device="cuda") for k in ("logprob", "coef")}
    report = rl.new_report()
    dh = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(V, H, device="cuda")
    adv = torch.empty(R, device="cuda")

    def step():
        rl.rl_group_advantages(d["rewards"], b.wl.group_size, adv)
        rl.rl_policy_loss_fwd_bwd(shape, params, d["hidden"], d["w"], d["targets"], d["infer"], adv, d["offsets"],
                                  d["loss_mask"], report=report, logprob=out["logprob"], coef=out["coef"],
                                  d_hidden=dh, d_w_vocab=dw, workspace=ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()                                   # warm-up (sets kernel attributes)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    # new inputs in the captured buffers, replay, and compare with an eager run
    d["hidden"].copy_(torch.roll(d["hidden"], 1, 0))
    g.replay()
    torch.cuda.synchronize()
    got = (out["logprob"].clone(), dh.clone(), dw.clone(), report.clone())
    step()
    torch.cuda.synchronize()
    for a, e in zip(got, (out["logprob"], dh, dw, report)):
        assert torch.equal(a, e)


# ---------------------------------------------- realistic rollouts
MID = synth.Workload("mid", 2, 8, 80, 512, 4184, ragged=True, prompt_frac=0.1, delta_sigma=0.5, spike_rate=2e-3)
# sigma_z = 32: 60% of the sampled targets at p_y > 0.99, a third at 1 - p_y < 1e-4
PEAKED = synth.Workload("peaked", 2, 8, 80, 512, 4184, sigma_z=32.0, ragged=True, delta_sigma=0.3, spike_rate=2e-3)
FLAT = synth.Workload("flat", 2, 8, 80, 512, 4184, sigma_z=1.0, ragged=True, delta_sigma=0.3, spike_rate=2e-3)


@pytest.mark.parametrize("wl", [MID, PEAKED, FLAT], ids=lambda w: w.name)
@pytest.mark.parametrize("dense", [False, True], ids=["sparse", "dense"])
def test_sampled_targets_and_band_plants(wl, dense):
    """Targets sampled from the policy itself (y ~ pi), guard spikes
    on the row's least likely token, and tokens planted at ln alpha, ln beta, ln tau_g
    +- {1e-6, 2e-4, 1e-3} (Eq.2, guard P:L472): outside the 1e-4 band the gate
    is exact. PEAKED (sigma_z = 32) puts most sampled targets at p_y > 0.99, where K4
    forms p - 1 by cancellation; FLAT (sigma_z = 1) is the high-entropy end."""
    c = harness.make_case(wl, 21, targets="sampled", plants=True)
    ref = harness.run_oracle(c)
    py = np.exp(ref.logp)
    if wl is PEAKED:
        assert np.mean(py > 0.99) > 0.5                       # the p_y -> 1 regime is exercised
    assert len(c.plants) >= 12 and ref.report.guarded_rollouts >= 1
    gpu = harness.run_gpu_step(c, dense_backward=dense)
    err = harness.compare(c, ref, gpu)
    print(wl.name, "dense" if dense else "sparse", {k: v for k, v in err.items()},
          "mean p_y", float(py.mean()), "plants", len(c.plants))
    assert err["plants_outside_band"] >= 8


# H = 8192 (a larger model's hidden size: 128 k-blocks per tile, twice GLM-4.5-Air's), a
# vocabulary that ends mid-tile (3001 = 11 * 256 + 185), sampled targets and band plants
WIDE_H = synth.Workload("wide-h", 2, 6, 50, 8192, 3001, ragged=True, delta_sigma=0.5, spike_rate=5e-3)


def test_hidden_8192_vs_oracle(monkeypatch):
    """Beyond the north star's GLM shape: the tensor cores' fp32 accumulation over 128
    k-blocks leaves logit errors of a few 1e-4 (about twice H = 4096's), more than the
    1e-4 band of the contract. Log-probs are held to 2e-3 as always; the gate may flip
    only where the row's OWN log-prob error can carry its ratio across a bound: the band
    is widened to beta * (the measured max log-prob error), the widest k-space image of
    a log-space error at the three bounds. Gradients given the gate as everywhere."""
    c = harness.make_case(WIDE_H, 22, targets="sampled", plants=True)
    ref = harness.run_oracle(c)
    for dense in (False, True):
        gpu = harness.run_gpu_step(c, dense_backward=dense)
        lp_err = float(np.max(np.abs(gpu["logprob"] - ref.logp)))
        assert lp_err <= harness.LOGP_TOL
        monkeypatch.setattr(harness, "BAND", max(harness.BAND, c.beta * lp_err * 1.01))
        c.plants = {}
        err = harness.compare(c, ref, gpu)
        print("H=8192", "dense" if dense else "sparse", "band", harness.BAND, err)
