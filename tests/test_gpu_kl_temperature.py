"""KL term (R19) and per-token temperature (R20) on the GPU vs the fp64 oracle (`-m gpu`).

Both change only S3's coefficient (KL) or the per-row logit scale (temperature), so
they ride through every backward path: dense and sparse, chunked dU buffers, the
three loss variants, and the vocab-parallel split phases."""
import numpy as np
import pytest

import harness
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_16144_b200 as rl  # noqa: E402

RAGGED = synth.Workload("ragged", 3, 4, 28, 200, 1000, ragged=True, prompt_frac=0.1, delta_sigma=0.8,
                        spike_rate=0.02)
T_TOK = 333


def _invt(seed):
    # fp32 values, handed to the oracle exactly as the GPU sees them
    return np.random.default_rng(seed).uniform(0.6, 1.6, T_TOK).astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("variant,kl_tau,kl_set,per_token,chunk,dense", [
    ("icepop", 0.3, "masked", False, 0, False),
    ("icepop", 0.3, "all", True, 0, False),
    ("icepop", 0.2, "unmasked", True, 100, False),
    ("icepop", 0.2, "masked", True, 128, True),
    ("cispo", 0.3, "unmasked", False, 0, False),
    ("gspo", 0.1, "masked", True, 0, False),
])
def test_kl_and_temperature_vs_oracle(variant, kl_tau, kl_set, per_token, chunk, dense):
    invT = _invt(1) if per_token else 1.0
    c = harness.make_case(RAGGED, 41, tokens=T_TOK, vocab=1000, hidden=392, inv_temperature=invT)
    c.variant, c.kl_tau, c.kl_set = variant, kl_tau, kl_set
    D = float(len(c.adv)) if variant == "gspo" else c.batch.loss_denominator
    ref = harness.run_oracle(c, loss_denominator=D)
    gpu = harness.run_gpu_step(c, loss_denominator=D, dz_chunk_rows=chunk, dense_backward=dense)
    err = harness.compare(c, ref, gpu)
    # the KL term moves the coefficient of the tokens outside the kept set too
    if kl_set == "masked":
        S = ref.report.valid & ~ref.report.keep
        band = harness.band_tokens(c, ref)
        sel = S & ~band & (gpu["keep"] == 0)
        np.testing.assert_allclose(gpu["coef"][sel], ref.report.coef[sel], rtol=1e-5, atol=0)
    print(err)


def test_per_token_temperature_constant_equals_scalar_bitwise():
    """A [T] array of one value gives the scalar path's outputs bit for bit."""
    c = harness.make_case(RAGGED, 42, tokens=T_TOK, vocab=1000, hidden=200, inv_temperature=1 / 0.7)
    g1 = harness.run_gpu_step(c)
    c.inv_temperature = np.full(T_TOK, np.float32(1 / 0.7), dtype=np.float64)
    g2 = harness.run_gpu_step(c)
    for k in ("logprob", "entropy", "lse", "coef", "d_hidden", "d_w_vocab"):
        assert np.array_equal(g1[k], g2[k]), k


def test_per_token_temperature_vocab_parallel_phases():
    """Three emulated vocab shards through the split-phase ABI with per-row 1/tau."""
    invT = _invt(3)
    c = harness.make_case(RAGGED, 43, tokens=T_TOK, vocab=1000, hidden=200, inv_temperature=invT)
    c.kl_tau = 0.25
    ref = harness.run_oracle(c)
    d = harness.to_device(c)
    b = c.batch
    T, H, V, R = b.T, b.H, b.V, len(c.adv)
    invt = torch.from_numpy(invT.astype(np.float32)).cuda()
    cuts = [0, 256, 600, 1000]
    parts = torch.empty(len(cuts) - 1, T, 4, device="cuda")
    for j, (a, e) in enumerate(zip(cuts[:-1], cuts[1:])):
        shp = rl.make_shape(T, H, e - a, a, V, inv_temperature_rows=invt)
        rl.rl_fwd_partials(shp, d["hidden"], d["w"][a:e].contiguous(), d["targets"], parts[j])
    lp, ent, lse = (torch.empty(T, device="cuda") for _ in range(3))
    rl.rl_merge_partials(parts, len(cuts) - 1, T, lp, ent, lse)
    coef = torch.empty(T, device="cuda")
    keep = torch.empty(T, dtype=torch.uint8, device="cuda")
    guarded = torch.empty(R, dtype=torch.uint8, device="cuda")
    report = rl.new_report()
    params = rl.make_params(R, b.loss_denominator, kl_tau=0.25)
    rl.rl_loss_coef(params, T, V, lp, d["infer"], d["targets"], d["adv"], d["offsets"], d["loss_mask"], coef,
                    keep, guarded, report=report)
    dh = torch.zeros(T, H, device="cuda")
    dws = []
    for a, e in zip(cuts[:-1], cuts[1:]):
        shp = rl.make_shape(T, H, e - a, a, V, inv_temperature_rows=invt)
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


def test_bad_kl_params_rejected():
    c = harness.make_case(RAGGED, 44, tokens=64, vocab=1000, hidden=64)
    c.kl_tau = float("nan")
    with pytest.raises(rl.RLError):
        harness.run_gpu_step(c)
    c.kl_tau, c.kl_set = 0.1, 7
    with pytest.raises(rl.RLError):
        harness.run_gpu_step(c)


def test_hostio_slabs_with_per_token_temperature():
    """The host-I/O call runs the forward slab by slab as the hidden rows arrive
    (slab ends 1024, 4096, ...); the per-row temperature pointer is offset per slab.
    Its outputs equal the device-resident call's bit for bit."""
    wl = synth.Workload("slab", 4, 4, 320, 64, 512, ragged=True, delta_sigma=0.8, spike_rate=0.001)
    T = 5000
    invT = np.random.default_rng(9).uniform(0.6, 1.6, T).astype(np.float32).astype(np.float64)
    c = harness.make_case(wl, 45, tokens=T, vocab=512, hidden=64, inv_temperature=invT)
    c.kl_tau = 0.125
    gdev = harness.run_gpu_step(c)
    b = c.batch
    H, V, R = b.H, b.V, len(c.adv)
    d = harness.to_device(c)
    invt = torch.from_numpy(invT.astype(np.float32)).cuda()
    shape = rl.make_shape(T, H, V, inv_temperature_rows=invt)
    params = rl.make_params(R, b.loss_denominator, kl_tau=0.125)
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
    harness.compare(c, harness.run_oracle(c), gdev)
