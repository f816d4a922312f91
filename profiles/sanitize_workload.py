"""Small workload for compute-sanitizer (race / sync / memory
checks of the hand-rolled mbarrier rings, shared-memory exchanges and fp64
shared atomics). One tool per gpurun call, e.g.

  compute-sanitizer --tool racecheck --error-exitcode 9 python profiles/sanitize_workload.py

Covers: the solver iteration at 128^3 (stencil2 TMA ring + s ring, z pass,
y / x passes, finalize) in audit + trace mode and FISTA; the TMA y pass and
the opt-in fused K1 cluster kernel at 256^3 (one iteration each); fft3_centered;
FSC of two resident results; device backprojection and E-step (dense and
sparse) at 16^3; a radix-5 side (40^3)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402
from paper_1905_13408_b200.backproject import GAUSSIAN  # noqa: E402


def solve(n, iters, **kw):
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, 32)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = cm.RegConfig(**{**cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime).__dict__,
                          "inner_iters": iters, **kw})
    ctx.set_volumes(p.x0, p.x0)
    tr = []
    ctx.solve(cfg, tr)
    x = ctx.get_volume()
    return ctx, x


ctx_a, xa = solve(128, 2)                                   # audit + trace, per_inner
ctx_b, xb = solve(128, 2, momentum=1, refresh=cm.Refresh.per_m_step)  # FISTA
curve = ctx_a.fsc(ctx_b)
V = ctx_a.get_spectrum(centered=True)
F = cm.fft3_centered(np.random.default_rng(0).standard_normal((40, 40, 40)))
ctx_a.close()
ctx_b.close()
solve(40, 2)                                                # radix-5 plan
solve(256, 1)                                               # TMA y pass
os.environ["CM_K1F"] = "1"
solve(256, 1)                                               # fused K1 (clusters, st.async)
os.environ.pop("CM_K1F")

inp = synth.synthetic_backprojection(16, 6, n_poses=7, trans_radius=1, kernel_kind=GAUSSIAN, seed=3)
ctx = cm.Context(16)
rng = np.random.default_rng(1)
Vs = rng.standard_normal((16, 16, 16)) + 1j * rng.standard_normal((16, 16, 16))
s2 = 16 * (1.0 + 0.05 * np.arange(9))
dense = cm.e_step(ctx, inp, s2, volume=Vs)
rows = cm.e_step(ctx, inp, s2, volume=Vs, sparse=True)
inp.entry_particle, inp.entry_candidate, inp.entry_posterior = cm.sparse_entries(*rows)
cm.backproject_into(ctx, inp)
ctx.close()
print("sanitize workload ok", float(curve[1]), float(np.abs(V).max()), float(np.abs(F).max()))
