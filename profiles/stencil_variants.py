"""Time the per-kernel profile of a 512^3 solve for the library in CM_LIBRARY
(variant comparison): python profiles/stencil_variants.py [iters]"""
import sys
sys.path.insert(0, ".")
import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 512
p = synth.synthetic_problem(n)
acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
ctx = cm.Context(n, 32)
ctx.set_accumulator(acc)
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = iters
ctx.set_volumes(p.x0, p.x0)
ctx.solve(cfg)
st = ctx.solve(cfg)
ctx.set_profiling(True)
ctx.solve(cfg)
ms, it = ctx.get_profile()
print({k: round(v / it, 4) for k, v in zip(ctx.PROFILE_KERNELS, ms)}, "graph ms/iter", st.solve_ms / iters)
