"""Backprojection throughput: cm_backproject on the device vs the reference
backproject_accumulate on all host cores (oracle/_ref, its own worker threads),
on the same synthetic ParticleSet / posterior rows / grid. Unit: (entry,
component) pairs per second -- one rotated frequency spread through its 27-tap
Gaussian window (backproject.cpp:43-70). Writes gpurun_out/backproject.json."""
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

n = int(os.environ.get("N", "128"))
m = int(os.environ.get("IMAGES", "2000"))
kind = int(os.environ.get("KIND", "0"))
inp = synth.synthetic_backprojection(n, m, n_poses=200, trans_radius=2, entries_per_image=5,
                                     kernel_kind=kind, seed=1)
ncomp = n * n
work = int((inp.entry_posterior > 0).sum()) * ncomp
ctx = cm.Context(n)
cm.backproject_into(ctx, inp, download=False)  # warm-up
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    cm.backproject_into(ctx, inp, download=False)
    ts.append(time.perf_counter() - t)
dev = min(ts)
cm.set_particles(ctx, inp)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    cm.backproject_into(ctx, inp, download=False, resident_images=True)
    ts.append(time.perf_counter() - t)
dev_res = min(ts)
res = {"device_s_resident_images": dev_res, "device_pairs_per_s_resident_images": work / dev_res,
       "n": n, "images": m, "kernel": ["gaussian", "trilinear"][kind],
       "entries_nonzero": int((inp.entry_posterior > 0).sum()), "components": ncomp,
       "device_s_incl_upload_and_commit": dev, "device_pairs_per_s": work / dev}
# reference on a bounded sample (first ms images), all host threads
from oracle_lib import Reference  # noqa: E402
ms = int(os.environ.get("REF_IMAGES", "100"))
sub = synth.synthetic_backprojection(n, ms, n_poses=200, trans_radius=2, entries_per_image=5,
                                     kernel_kind=kind, seed=1)
threads = os.cpu_count()
R = Reference()
t = time.perf_counter()
rc, w_ref, y_ref = R.backproject(sub, threads=threads)
tr = time.perf_counter() - t
assert rc == 0
sw = int((sub.entry_posterior > 0).sum()) * ncomp
acc = cm.backproject_accumulate(sub)
res.update({"reference_images": ms, "reference_threads": threads, "reference_s": tr,
            "reference_pairs_per_s": sw / tr,
            "speedup": (work / dev) / (sw / tr),
            "max_rel_err_numerator": float(np.abs(acc.numerator - y_ref).max() / np.abs(y_ref).max()),
            "max_rel_err_weight": float(np.abs(acc.weight - w_ref).max() / w_ref.max())})
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/backproject.json", "w"), indent=1)
