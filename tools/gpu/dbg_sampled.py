import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import harness, synth, oracle, numpy as np, torch
import paper_2512_16144_b200 as rl
MID = synth.Workload("mid", 2, 8, 80, 512, 4184, ragged=True, prompt_frac=0.1, delta_sigma=0.5, spike_rate=2e-3)
c = harness.make_case(MID, 21, targets="sampled", plants=True)
ref = harness.run_oracle(c)
for k0 in (False, True):
    g = harness.run_gpu_step(c, k0=k0)
    print("k0", k0, "loss", g["report"]["loss"], "ref", ref.report.loss)
    print(" guarded gpu", g["guarded"].astype(int), "\n guarded ref", ref.report.guarded.astype(int))
    fl = np.nonzero(g["keep"].astype(bool) != ref.report.keep)[0]
    print(" flips", len(fl), fl[:20], "coef diff max", np.abs(g["coef"]-ref.report.coef).max())
    print(" report", g["report"])
    print(" ref counters", ref.report.masked_low, ref.report.masked_high, ref.report.guarded_rollouts, ref.report.kept_tokens)
d = harness.to_device(c)
adv = rl.rl_group_advantages(d["rewards"], c.batch.rewards.shape[1])
print("adv gpu", adv.cpu().numpy(), "\nadv ref", c.adv)
