"""Host <-> device transfer rates of the drop-in's pageable buffers through the
pinned chunk ring (host_xfer.h) vs page-locked buffers: cm_m_step with
inner_iters = 1 at n^3 (so the transfers dominate), CM_XFER_THREADS set by the
caller. python profiles/xfer_bench.py [n]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = synth.synthetic_problem(n)
acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
ctx = cm.Context(n, 32)
ctx.set_accumulator(acc)
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = 1
out = np.empty((n, n, n))
ctx.m_step_host(acc, p.x0, p.x0, cfg, out)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    st = ctx.m_step_host(acc, p.x0, p.x0, cfg, out)
    ts.append(time.perf_counter() - t0 - st.solve_ms / 1e3)
L = n ** 3
print(json.dumps({"n": n, "bytes": 40 * L, "transfer_s": min(ts), "GBps": 40 * L / min(ts) / 1e9}))
