"""Small fixed workload for ncu captures: one resident 512^3 problem, a short
solve through the C ABI (same kernels as bench.py). Usage:
  python profiles/profile_step.py [n] [iters] [precision]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 32
p = synth.synthetic_problem(n)
ctx = cm.Context(n, prec)
ctx.set_accumulator(cm.AccumulatorPair(n, p.numerator, p.weight, True))
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = iters
if len(sys.argv) > 4:  # timing experiments: never stop on the audit
    cfg.audit_slack = float(sys.argv[4])
ctx.set_volumes(p.x0, p.x0)
ctx.set_profiling(True)  # one launch per kernel (no graph) so ncu sees each
try:
    st = ctx.solve(cfg)
    print("iterations", st.iterations, "solve_ms", st.solve_ms, "profile", ctx.get_profile())
except cm.Error as e:  # timing experiments may produce garbage iterates
    print("error", type(e).__name__, "profile", ctx.get_profile())
