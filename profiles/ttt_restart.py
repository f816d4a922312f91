"""FISTA with and without gradient-based adaptive restart (momentum 1 / 2) at
n^3: iterations, seconds and error against the converged frozen-weight
solution, for the step-norm rule (tol_kind 2). Writes one JSON object.

  python profiles/ttt_restart.py [n] [ref_iters] > profiles/r2_ttt_restart.json"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ref_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12000
p = synth.synthetic_problem(n)
ctx = cm.Context(n, 32)
ctx.set_accumulator(cm.AccumulatorPair(n, p.numerator, p.weight, True))
s = ctx.scale_data()
base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
ctx.set_volumes(p.x0, p.x0)


def solve(**kw):
    st = ctx.solve(cm.RegConfig(**{**base.__dict__, "refresh": cm.Refresh.per_m_step, **kw}))
    return ctx.get_volume(), st


xs, _ = solve(inner_iters=ref_iters, momentum=1)
nx = float(np.linalg.norm(xs))
out = {"n": n, "reference_solution": f"FISTA, {ref_iters} iterations, per_m_step", "runs": []}
for mom in (1, 2):
    for tol in (0.1, 0.03, 0.01):
        x, st = solve(inner_iters=ref_iters, momentum=mom, tol_kind=2, tol=tol)
        out["runs"].append({"momentum": mom, "tol": tol, "iterations": st.iterations,
                            "seconds": st.solve_ms / 1e3,
                            "rel_err": float(np.linalg.norm(x - xs)) / nx})
        print(out["runs"][-1], file=sys.stderr)
print(json.dumps(out, indent=1))
