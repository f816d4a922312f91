"""A/B of run-time kernel switches on one 512^3 (or n^3) solve.

  python profiles/ab_env.py [n] [iters] VAR=a,b [VAR2=c,d ...]

Runs, for every combination of the listed environment values, a child process
that builds the solver context under that environment, times the per-iteration
kernels (CUDA events, profiling solve) and the graph-replayed solve, and saves
the result volume; prints one JSON line per variant plus the relative L2
difference of each variant's volume against the first (the switches must not
change results beyond fp32 roundoff). AB_PREC=64 in the environment (or as a
switch) runs the fp64 parity mode."""
import itertools
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, ".")
import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
n, iters, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
p = synth.synthetic_problem(n)
acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
import os
ctx = cm.Context(n, int(os.environ.get("AB_PREC", "32")))
ctx.set_accumulator(acc)
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = iters
ctx.set_volumes(p.x0, p.x0)
ctx.solve(cfg)
best = min(ctx.solve(cfg).solve_ms for _ in range(3)) / iters
x = ctx.get_volume()
ctx.set_profiling(True)
ctx.solve(cfg)
ms, it = ctx.get_profile()
np.save(out, x)
print(json.dumps({"kernels_ms": {k: round(v / it, 4) for k, v in zip(ctx.PROFILE_KERNELS, ms)},
                  "graph_ms_per_iter": round(best, 4)}))
"""


def main():
    n = int(sys.argv[1])
    iters = int(sys.argv[2])
    axes = []
    for a in sys.argv[3:]:
        k, v = a.split("=", 1)
        axes.append([(k, x) for x in v.split(",")])
    ref = None
    with tempfile.TemporaryDirectory() as td:
        for combo in itertools.product(*axes):
            env = dict(os.environ, **dict(combo))
            out = os.path.join(td, "x.npy")
            r = subprocess.run([sys.executable, "-c", CHILD, str(n), str(iters), out], env=env,
                               capture_output=True, text=True)
            if r.returncode != 0:
                print(json.dumps({"env": dict(combo), "error": r.stderr[-1500:]}), flush=True)
                continue
            line = json.loads(r.stdout.strip().splitlines()[-1])
            x = np.load(out).astype(np.float64)
            if ref is None:
                ref = x
            line["env"] = dict(combo)
            line["rel_l2_vs_first"] = float(np.linalg.norm(x - ref) / np.linalg.norm(ref))
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
