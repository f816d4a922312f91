"""Times cm_write_volume_mrc / cm_set_volumes_mrc at 512^3 against the
double-precision host path a reference user takes (get_volume + write of the
float32 payload; read + set_volumes). Writes gpurun_out/mrc_io.json."""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

n = int(os.environ.get("N", "512"))
p = synth.synthetic_problem(n)
acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
s = cm.scale_data(acc)
cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
cfg.inner_iters = 2
ctx = cm.Context(n)
ctx.set_accumulator(acc)
ctx.set_volumes(p.x0)
ctx.solve(cfg)
d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
f = os.path.join(d, "v.mrc")
res = {"n": n, "payload_bytes": 4 * n ** 3, "dir": d}
for rep in range(3):
    t = time.perf_counter(); ctx.write_volume_mrc(f, 1.0); tw = time.perf_counter() - t
    t = time.perf_counter(); ctx.set_volumes_mrc(f); tr = time.perf_counter() - t
    t = time.perf_counter()
    x = ctx.get_volume()
    with open(f + ".host", "wb") as fh:
        fh.write(b"\0" * 1024); fh.write(x.astype("<f4").tobytes())
    th_w = time.perf_counter() - t
    t = time.perf_counter()
    y = np.fromfile(f + ".host", "<f4", offset=1024).astype(np.float64)
    ctx.set_volumes(y.reshape(n, n, n))
    th_r = time.perf_counter() - t
    res[f"rep{rep}"] = dict(write_s=tw, read_s=tr, host_path_write_s=th_w, host_path_read_s=th_r)
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/mrc_io.json", "w"), indent=1)
