"""Per-kernel profile (CUDA events, profiling solve) of an n^3 solve at a given
precision: python profiles/prof_prec.py n precision iters"""
import json
import sys

sys.path.insert(0, ".")
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n, prec, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = synth.synthetic_problem(n)
ctx = cm.Context(n, prec)
ctx.set_accumulator(cm.AccumulatorPair(n, p.numerator, p.weight, True))
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = iters
ctx.set_volumes(p.x0, p.x0)
ctx.solve(cfg)
g = ctx.solve(cfg).solve_ms / iters
ctx.set_profiling(True)
ctx.solve(cfg)
ms, it = ctx.get_profile()
print(json.dumps({"n": n, "precision": prec, "graph_ms_per_iter": g,
                  "kernels_ms": {k: round(v / it, 4) for k, v in zip(ctx.PROFILE_KERNELS, ms)}}))
