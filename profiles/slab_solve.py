"""Run a device-rendered z-slab solve (profiling driver): python profiles/slab_solve.py N WORLD ITERS"""
import sys
sys.path.insert(0, ".")
import paper_1905_13408_b200 as cm
from paper_1905_13408_b200.slab import SlabContext
n = int(sys.argv[1]); world = int(sys.argv[2]); iters = int(sys.argv[3])
sc = SlabContext(n, world)
sy = sc.set_synthetic(7)
cfg = cm.derive_config(sy, 1.5, 0.1, 0.1 / 3)
cfg.inner_iters = iters
st = sc.solve(cfg)
print(st)
