"""Golden fixtures at the BASELINE.json sizes, from the UNMODIFIED reference.

Run here (where /root/reference exists):
    CM_REF_FFT_THREADS=8 python tests/golden/make_golden_baseline.py [--skip-512]

It drives oracle/_ref/libcryomap_ref.so (reference sources + the FFTW-API shim
over oneMKL, oracle/Makefile) on the synthetic inputs of SURVEY §8(d)
(paper_1905_13408_b200.synth, pure functions of seeds) and records:

  config 1  64^3 blob phantom, 100 iterations, ONE m_step call, refresh
            per_m_step (single reweighting pass), lipschitz step + audit — the
            configuration exactly as BASELINE.json names it; plus the same with
            the reference's default per_inner refresh. Full trace rows
            (before/after ObjectiveValue + step, regularizer.cpp:215) and x.
  config 2  256^3 bond-like (chain) phantom, three reweighting loops: m_step
            calls with per_m_step refresh, x_init <- previous output, anchor =
            the initial volume (refine.cpp:181 pattern), 4 iterations each;
            plus one per_inner call of 6 iterations. Trace rows, ||x||_2 and x
            at a fixed random sample of voxels (the npz stays small).
  config 3  512^3 blob phantom, reference default semantics (lipschitz, audit,
            per_inner), 2 iterations: trace rows, ||x||_2 and a voxel sample.

CM_REF_FFT_THREADS only sets the FFT backend's thread count (results agree to
roundoff). Inputs are not stored: each entry carries the sha256 of its inputs
so the GPU test proves it fed the same bytes.
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from golden.make_golden import sha  # noqa: E402
from oracle_lib import Reference, build_oracles, make_cfg  # noqa: E402
from paper_1905_13408_b200 import synth  # noqa: E402

OUT = HERE / "reference_baseline.npz"
NSAMPLE = 65536


def sample_index(n: int) -> np.ndarray:
    """The fixed voxel sample (flat x-fastest indices) stored for n >= 256."""
    return np.sort(np.random.default_rng(1234 + n).choice(n ** 3, NSAMPLE, replace=False))


def cfg_of(R, p, iters, **extra):
    rc, sy, sn = R.scale_data(p.weight, p.numerator)
    assert rc == 0, R.last_error()
    rc, base = R.derive_config(sy, sn, p.eps, p.eps_prime)
    assert rc == 0, R.last_error()
    c = make_cfg(alpha=base.alpha, beta=base.beta, gamma=base.gamma, eps=base.eps,
                 eps_prime=base.eps_prime, mu=base.mu, inner_iters=iters)
    for k, v in extra.items():
        setattr(c, k, v)
    return c, np.array([sy, sn])


def run(R, p, x_init, c, key, out, full_x: bool):
    t0 = time.time()
    rc, x, tr = R.m_step(p.weight, p.numerator, x_init, p.x0, c, trace=True)
    assert rc == 0, R.last_error()
    out[key + "_trace"] = tr
    out[key + "_norm"] = np.array([np.linalg.norm(x)])
    if full_x:
        out[key + "_x"] = x.astype(np.float32)
    else:
        out[key + "_xsample"] = x.reshape(-1)[sample_index(p.n)]
    print(f"  {key}: {c.inner_iters} iterations in {time.time() - t0:.1f} s", flush=True)
    return x


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-512", action="store_true")
    a = ap.parse_args()
    build_oracles()
    R = Reference()
    out = {}

    # ---- config 1: 64^3, 100 iterations, one reweighting pass
    p = synth.synthetic_problem(64)
    out["c1_sha"] = sha(p.weight, p.numerator, p.x0)
    for name, extra in (("per_m_step", dict(refresh=1)), ("per_inner", dict())):
        c, scales = cfg_of(R, p, 100, **extra)
        out["c1_scales"] = scales
        run(R, p, p.x0, c, f"c1_{name}", out, full_x=True)

    # ---- config 2: 256^3 chains, three per_m_step loops of 4 + one per_inner call
    p = synth.synthetic_problem(256, kind="bonds")
    out["c2_sha"] = sha(p.weight, p.numerator, p.x0)
    c, scales = cfg_of(R, p, 4, refresh=1)
    out["c2_scales"] = scales
    x = p.x0
    for loop in range(3):
        x = run(R, p, x, c, f"c2_loop{loop}", out, full_x=False)
    c, _ = cfg_of(R, p, 6)
    run(R, p, p.x0, c, "c2_per_inner", out, full_x=False)
    del p, x

    # ---- config 3: 512^3, reference defaults, 2 iterations
    if not a.skip_512:
        p = synth.synthetic_problem(512)
        out["c3_sha"] = sha(p.weight, p.numerator, p.x0)
        c, scales = cfg_of(R, p, 2)
        out["c3_scales"] = scales
        run(R, p, p.x0, c, "c3_per_inner", out, full_x=False)

    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
