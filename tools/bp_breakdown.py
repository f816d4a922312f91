"""Per-stage host-clock breakdown of the device EM iteration's E-step and
backprojection at 128^3 (bench.em_iteration's shapes)."""
import time, json, numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
n, m = 128, 1000
inp = synth.synthetic_backprojection(n, m, n_poses=200, trans_radius=2, entries_per_image=3, seed=11)
sigma2 = np.ones(n // 2 + 1)
ctx = cm.Context(n, 32, device=0)
cm.set_particles(ctx, inp)
cm.backproject_into(ctx, inp, download=False, resident_images=True)
s = ctx.scale_data()
cfg = cm.derive_config(s.s_y, s.s_n, 1e-3, 1e-3)
cfg.inner_iters = 50
x = np.zeros((n, n, n)); ctx.set_volumes(x)
ctx.solve(cfg)
for r in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    post = cm.e_step(ctx, inp, sigma2, resident_images=True)
    t1 = time.perf_counter()
    inp.entry_particle, inp.entry_candidate, inp.entry_posterior = cm.posterior_entries(post)
    t2 = time.perf_counter()
    c = inp.to_c(True)
    t3 = time.perf_counter()
    cm.backproject_into(ctx, inp, download=False, resident_images=True)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    cm.backproject_into(ctx, inp, download=False, resident_images=True)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(json.dumps(dict(estep=t1-t0, entries=t2-t1, to_c=t3-t2, bp=t4-t3, bp_again=t5-t4, n=int(inp.entry_posterior.size))), flush=True)
