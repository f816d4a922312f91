"""E-step throughput: cm_estep on the device vs the reference e_step on all
host cores (oracle/_ref, its own worker threads), same synthetic particles,
volume, grid and noise spectrum. Unit: (particle, pose) pairs per second
(each: a pass-1 sweep over the components, plus all shifts when the pose
survives the bound). Writes gpurun_out/estep.json."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1905_13408_b200 as cm  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402
from oracle_lib import Reference  # noqa: E402

n = int(os.environ.get("N", "128"))
m = int(os.environ.get("IMAGES", "1000"))
npose = int(os.environ.get("POSES", "200"))
scale = float(os.environ.get("SCALE", "1.0"))


def problem(m_):
    inp = synth.synthetic_backprojection(n, m_, n_poses=npose, trans_radius=2, seed=2)
    rng = np.random.default_rng(7)
    V = rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n))
    s2 = scale * n * (1.0 + 0.05 * np.arange(n // 2 + 1))
    return inp, V, s2


inp, V, s2 = problem(m)
ctx = cm.Context(n)
cm.e_step(ctx, inp, s2, volume=V)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    post = cm.e_step(ctx, inp, s2, volume=V)
    ts.append(time.perf_counter() - t)
dev = min(ts)
cm.set_particles(ctx, inp)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    cm.e_step(ctx, inp, s2, volume=V, resident_images=True)
    ts.append(time.perf_counter() - t)
dev_res = min(ts)
res = {"device_s_resident_images": dev_res, "device_pairs_per_s_resident_images": m * npose / dev_res,
       "n": n, "images": m, "poses": npose, "shifts": int(inp.shifts.shape[0]),
       "device_s_incl_transfers": dev, "device_pairs_per_s": m * npose / dev,
       "mean_entries_per_row": float((post > 0).sum(axis=1).mean())}
ms = int(os.environ.get("REF_IMAGES", "64"))
sub, V2, _ = problem(ms)
R = Reference()
threads = os.cpu_count()
t = time.perf_counter()
rc, want = R.estep(sub, V2, s2, threads=threads)
tr = time.perf_counter() - t
assert rc == 0
got = cm.e_step(ctx, sub, s2, volume=V2)
res.update({"reference_images": ms, "reference_threads": threads, "reference_s": tr,
            "reference_pairs_per_s": ms * npose / tr,
            "speedup": (m * npose / dev) / (ms * npose / tr),
            "max_abs_err": float(np.abs(got - want).max()),
            "support_equal": bool(((got != 0) == (want != 0)).all())})
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/estep.json", "w"), indent=1)
