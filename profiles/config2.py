"""BASELINE config 2 on one B200: 256^3 bond-like (chain) phantom, three m_step
calls with per_m_step reweighting (x_init <- previous output, anchor fixed at the
initial volume), each run to tolerance. Writes one JSON line.

  python profiles/config2.py [n] > profiles/r1_config2_256.json

Tolerances: ISTA (the reference's update) stops on the frozen-weight surrogate
relative decrease < 1e-6 (SURVEY §8(d) config 3 proposal), capped at 20000
iterations; FISTA (opt-in) on the step-norm rule at 3% (the rule calibrated at
512^3 in r1_convergence_512.json)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t0 = time.time()
p = synth.synthetic_problem(n, kind="bonds")
gen = time.time() - t0
acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
ctx = cm.Context(n, 32)
ctx.set_accumulator(acc)
s = ctx.scale_data()
base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
out = {"config": f"BASELINE config 2: {n}^3 bond-like phantom, 3 reweighting loops "
                  "(per_m_step, x_init <- previous output, anchor = initial)",
       "gen_seconds": gen, "runs": {}}
for name, extra in (("ista_surrogate_1e-6", dict(tol_kind=1, tol=1e-6)),
                    ("fista_step_3pct", dict(momentum=1, tol_kind=2, tol=0.03))):
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 20000,
                          "refresh": cm.Refresh.per_m_step, **extra})
    x = p.x0
    loops = []
    for loop in range(3):
        ctx.set_volumes(x, p.x0)
        st = ctx.solve(cfg)
        x = ctx.get_volume()
        loops.append({"iterations": st.iterations, "seconds": st.solve_ms / 1e3,
                      "stop_reason": st.stop_reason, "last_rel": st.last_rel})
    err = float(np.linalg.norm(x - p.truth) / np.linalg.norm(p.truth))
    out["runs"][name] = {"loops": loops, "total_seconds": sum(l["seconds"] for l in loops),
                         "rel_err_vs_truth": err}
print(json.dumps(out))
