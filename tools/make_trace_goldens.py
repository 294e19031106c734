"""Writes tests/golden/trace_cond.json: for each config, the oracle's replayed phase schedule and
the conditioning of its 20-sweep trace (tests/trace_check.py: the drift between the oracle run
and oracle runs from initial factors moved by one ulp).  Calls only oracle/ and synthgen/.

  python tools/make_trace_goldens.py [C1 C2mini ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synthgen as G  # noqa: E402
from trace_check import GOLDEN, conditioning  # noqa: E402

DEFAULT = ["C1", "C2mini", "C3mini", "C4mini", "C5mini", "LAPmini", "C2", "C3", "C4"]


def main():
    names = sys.argv[1:] or DEFAULT
    out = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}
    for name in names:
        cfg = G.CONFIGS[name]
        t0 = time.time()
        X = G.make_tensor(cfg)
        A0 = G.initial_factors(cfg)
        c = conditioning(X, A0, cfg.eps_pp, cfg.sweeps)
        c["config"] = name
        c["note"] = ("oracle/cp_oracle.py pp_cp_als, 0 global stop, eps_pp %g, %d sweeps; delta = drift "
                     "to one-ulp perturbed initial factors (both directions), running max" % (cfg.eps_pp, cfg.sweeps))
        out[name] = c
        print(name, "%.1fs" % (time.time() - t0), {q: "%.1e" % v[-1] for q, v in c["delta"].items()},
              "dA %.1e" % c["delta_factors"], flush=True)
        with open(GOLDEN, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
