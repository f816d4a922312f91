"""Convergence study for "time to tolerance" (open question 1).

The reference has no stopping rule; the paper claims a "medium accurate
solution". We measure accuracy directly: a long FISTA run with
frozen weights (per_m_step, a convex subproblem) gives x*; ISTA (the
reference's method) and FISTA are then run for k iterations from x0 and scored
by ||x_k - x*|| / ||x*|| and the frozen-weight surrogate gap.

  python profiles/convergence.py [n] [ref_iters] > profiles/convergence_<n>.json
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ref_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
t0 = time.time()
p = synth.synthetic_problem(n)
ctx = cm.Context(n, 32)
ctx.set_accumulator(cm.AccumulatorPair(n, p.numerator, p.weight, True))
s = ctx.scale_data()
base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
base.refresh = cm.Refresh.per_m_step
ctx.set_volumes(p.x0, p.x0)


def run(iters, momentum):
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": iters, "momentum": momentum,
                          "step_rule": cm.StepRule.lipschitz})
    st = ctx.solve(cfg)
    return ctx.get_volume(), st


xs, st = run(ref_iters, 1)
nref = float(np.linalg.norm(xs))
out = {"n": n, "ref": {"method": "fista", "iters": ref_iters, "seconds": st.solve_ms / 1e3},
       "config": {k: (float(v) if isinstance(v, float) else int(v)) for k, v in base.__dict__.items()},
       "ista": [], "fista": []}
for name, mom, ks in (("ista", 0, [50, 100, 200, 500, 1000, 2000, 4000, 8000]),
                      ("fista", 1, [25, 50, 100, 200, 400, 800, 1600, 3200])):
    for k in ks:
        x, st = run(k, mom)
        out[name].append({"iters": k, "rel_err": float(np.linalg.norm(x - xs)) / nref,
                          "ms": st.solve_ms, "ms_per_iter": st.solve_ms / k})
    print(name, [(r["iters"], round(r["rel_err"], 6)) for r in out[name]], file=sys.stderr)
# practical stopping rules (no x* at run time): where do they stop, how accurate?
out["stops"] = []
for name, mom, kind, taus in (("fista", 1, 2, [3e-2, 1e-2, 3e-3, 1e-3, 3e-4]),
                              ("ista", 0, 1, [1e-5, 3e-6, 1e-6, 3e-7])):
    for tau in taus:
        cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 20000, "momentum": mom,
                              "tol_kind": kind, "tol": tau})
        st = ctx.solve(cfg)
        x = ctx.get_volume()
        out["stops"].append({"method": name, "criterion": "step norm / largest step" if kind == 2 else
                             "surrogate relative decrease", "tol": tau, "iters": st.iterations,
                             "seconds": st.solve_ms / 1e3,
                             "rel_err": float(np.linalg.norm(x - xs)) / nref})
        print(out["stops"][-1], file=sys.stderr)
out["wall_s"] = time.time() - t0
print(json.dumps(out, indent=1))
