"""Write one input artifact (synth/artifact.py) plus the fp64 oracle's
outputs next to it, so a GPU process can be checked against the oracle without the two
ever running in the same process.

    python tests/make_artifact.py --config tiny --seed 0 --out DIR [--tokens T --vocab V --hidden H]
                                  [--targets sampled|uniform] [--plants]

Inputs come from `harness.make_case` (seeded synth draws; sampled targets and the stored
inference log-probs composed from the oracle's own log-probs). Outputs (oracle only):
oracle_{logprob,entropy,lse,ratio,coef,keep,valid,guarded,d_hidden,d_w_vocab}.npy and
oracle_report.json. Test infrastructure: calls nothing but `oracle/` and `synth/`.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import harness  # noqa: E402
import synth  # noqa: E402
from synth import artifact  # noqa: E402


def write_case(out: str, c: harness.Case, targets: str) -> dict:
    meta = artifact.write(out, c.batch, c.infer, alpha=c.alpha, beta=c.beta, guard=c.guard,
                          inv_temperature=float(c.inv_temperature), targets=targets)
    ref = harness.run_oracle(c)
    r = ref.report
    for name, arr in (("logprob", ref.logp), ("entropy", ref.entropy), ("lse", ref.lse), ("ratio", r.ratio),
                      ("coef", r.coef), ("keep", r.keep), ("valid", r.valid), ("guarded", r.guarded),
                      ("d_hidden", ref.d_hidden), ("d_w_vocab", ref.d_w_vocab), ("advantages", c.adv)):
        np.save(os.path.join(out, f"oracle_{name}.npy"), np.asarray(arr))
    rep = {k: (float(getattr(r, k)) if k in ("loss", "mismatch_kl_sum") else int(getattr(r, k)))
           for k in ("loss", "mismatch_kl_sum", "kept_tokens", "masked_low", "masked_high", "guarded_tokens",
                     "guarded_rollouts", "nonfinite_inputs", "bad_targets", "bad_offsets")}
    rep["plants"] = {str(k): list(v) for k, v in c.plants.items()}
    with open(os.path.join(out, "oracle_report.json"), "w") as f:
        json.dump(rep, f, indent=1, sort_keys=True)
    return meta


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny", choices=sorted(synth.CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--tokens", type=int)
    ap.add_argument("--vocab", type=int)
    ap.add_argument("--hidden", type=int)
    ap.add_argument("--targets", default="sampled", choices=["sampled", "uniform"])
    ap.add_argument("--plants", action="store_true")
    a = ap.parse_args(argv)
    c = harness.make_case(synth.CONFIGS[a.config], a.seed, tokens=a.tokens, vocab=a.vocab, hidden=a.hidden,
                          targets=a.targets, plants=a.plants)
    meta = write_case(a.out, c, a.targets)
    print(json.dumps({"out": a.out, "T": meta["T"], "H": meta["H"], "V": meta["V"]}))


if __name__ == "__main__":
    main()
