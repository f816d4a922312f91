"""Debug helper: the sweep-mode sequence of tests/test_gpu_parity.py::
test_sweep_tiles_and_modes_vs_oracle for one (n, precision), printing each mode."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from test_gpu_parity import SWEEP_MODES, acc_of, random_volume

n = int(sys.argv[1]); prec = int(sys.argv[2])
if len(sys.argv) > 3:
    from oracle_lib import Oracle
    O = Oracle()  # the checker library loaded as in the pytest module
p = synth.synthetic_problem(n)
acc = acc_of(p.weight, p.numerator)
s = cm.scale_data(acc, precision=prec)
base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
anchor = p.x0 + 0.01 * random_volume(n, 99)
lr0 = 1.0 / (2.0 * p.weight.max() + 2.0 * base.gamma + 12.0 * base.beta / base.eps_prime / base.mu)
for name, extra in SWEEP_MODES.items():
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 8, "fixed_step": 2.0 * lr0, **extra})
    tr = []
    try:
        x = cm.m_step(acc, p.x0, anchor, cfg, tr, precision=prec)
        print(name, "ok", float(np.linalg.norm(x)), flush=True)
    except Exception as e:
        print(name, "FAIL", e, flush=True)
        break
