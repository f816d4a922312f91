"""Parity at the BASELINE.json sizes against the UNMODIFIED reference
(fixtures tests/golden/reference_baseline.npz, written by
tests/golden/make_golden_baseline.py from oracle/_ref/libcryomap_ref.so).

Bar (BASELINE.json north_star, fp32 product mode): every per-iteration
ObjectiveValue field within 1e-5 relative (relative to max(|field|,
|surrogate|), as tests/test_gpu_parity.py::check_trace) and the final volume
within 1e-4 relative L2 — on the full volume at 64^3, on a fixed 65536-voxel
sample plus ||x||_2 at 256^3 / 512^3. fp64 mode: 1e-9.

  config 1  64^3, 100 iterations, one m_step call, per_m_step (+ per_inner)
  config 2  256^3 chain phantom, three per_m_step loops (x_init <- previous
            output, anchor = initial; each loop's GPU start is the GPU's own
            previous output, so the chain is judged end to end) + per_inner
  config 3  512^3, reference default semantics, first 2 iterations
"""
from pathlib import Path

import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from golden.make_golden import sha
from golden.make_golden_baseline import sample_index

pytestmark = pytest.mark.gpu

GB = Path(__file__).parent / "golden" / "reference_baseline.npz"
G = np.load(GB) if GB.exists() else None
need = pytest.mark.skipif(G is None, reason="reference_baseline.npz not generated")
TOL = {32: dict(obj=1e-5, vol=1e-4), 64: dict(obj=1e-9, vol=1e-9)}


def check_trace(rows, ref, tol):
    got = np.array([np.r_[r.before.as_array(), r.after.as_array(), r.step] for r in rows])
    assert got.shape == ref.shape, (got.shape, ref.shape)
    worst = 0.0
    for half in (slice(0, 7), slice(7, 14)):
        g, r = got[:, half], ref[:, half]
        surr = np.abs(r[:, 0] + r[:, 1] + r[:, 2] + r[:, 4])
        err = np.abs(g - r) / np.maximum(np.abs(r), surr[:, None])
        worst = max(worst, float(err.max()))
        assert err.max() <= tol, (half, err.max(), np.unravel_index(err.argmax(), err.shape))
    np.testing.assert_allclose(got[:, 14], ref[:, 14], rtol=1e-12)
    return worst


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def config_of(ctx, p, key, iters, refresh):
    s = ctx.scale_data()
    np.testing.assert_allclose([s.s_y, s.s_n], G[key + "_scales"], rtol=1e-12)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = iters
    cfg.refresh = refresh
    return cfg


@need
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("mode", ["per_m_step", "per_inner"])
def test_config1_64cubed_100_iterations_vs_reference(prec, mode):
    p = synth.synthetic_problem(64)
    assert sha(p.weight, p.numerator, p.x0) == str(G["c1_sha"])
    ctx = cm.Context(64, prec)
    ctx.set_accumulator(cm.AccumulatorPair(64, p.numerator, p.weight, True))
    refresh = cm.Refresh.per_m_step if mode == "per_m_step" else cm.Refresh.per_inner
    cfg = config_of(ctx, p, "c1", 100, refresh)
    ctx.set_volumes(p.x0, p.x0)
    trace = []
    ctx.solve(cfg, trace)
    x = ctx.get_volume()
    ctx.close()
    check_trace(trace, G[f"c1_{mode}_trace"], TOL[prec]["obj"])
    # the fixture stores x in fp32 (relative precision 6e-8)
    assert rel(x, G[f"c1_{mode}_x"].astype(np.float64)) <= max(TOL[prec]["vol"], 1e-7)


@pytest.fixture(scope="module")
def bonds256():
    if G is None:
        pytest.skip("reference_baseline.npz not generated")
    p = synth.synthetic_problem(256, kind="bonds")
    assert sha(p.weight, p.numerator, p.x0) == str(G["c2_sha"])
    return p


@need
@pytest.mark.parametrize("prec", [32, 64])
def test_config2_256cubed_reweighting_loops_vs_reference(bonds256, prec):
    p = bonds256
    idx = sample_index(256)
    ctx = cm.Context(256, prec)
    ctx.set_accumulator(cm.AccumulatorPair(256, p.numerator, p.weight, True))
    cfg = config_of(ctx, p, "c2", 4, cm.Refresh.per_m_step)
    x = p.x0
    for loop in range(3):
        trace = []
        ctx.set_volumes(x, p.x0)
        ctx.solve(cfg, trace)
        x = ctx.get_volume()
        check_trace(trace, G[f"c2_loop{loop}_trace"], TOL[prec]["obj"])
        assert rel(x.reshape(-1)[idx], G[f"c2_loop{loop}_xsample"]) <= TOL[prec]["vol"], loop
        assert abs(np.linalg.norm(x) / G[f"c2_loop{loop}_norm"][0] - 1) <= TOL[prec]["vol"] / 10
    cfg = config_of(ctx, p, "c2", 6, cm.Refresh.per_inner)
    trace = []
    ctx.set_volumes(p.x0, p.x0)
    ctx.solve(cfg, trace)
    x = ctx.get_volume()
    ctx.close()
    check_trace(trace, G["c2_per_inner_trace"], TOL[prec]["obj"])
    assert rel(x.reshape(-1)[idx], G["c2_per_inner_xsample"]) <= TOL[prec]["vol"]


@need
def test_config3_512cubed_first_iterations_vs_reference():
    if "c3_sha" not in G.files:
        pytest.skip("512^3 fixture not generated")
    p = synth.synthetic_problem(512)
    assert sha(p.weight, p.numerator, p.x0) == str(G["c3_sha"])
    ctx = cm.Context(512, 32)
    ctx.set_accumulator(cm.AccumulatorPair(512, p.numerator, p.weight, True))
    cfg = config_of(ctx, p, "c3", 2, cm.Refresh.per_inner)
    ctx.set_volumes(p.x0, p.x0)
    trace = []
    ctx.solve(cfg, trace)
    x = ctx.get_volume()
    ctx.close()
    check_trace(trace, G["c3_per_inner_trace"], TOL[32]["obj"])
    assert rel(x.reshape(-1)[sample_index(512)], G["c3_per_inner_xsample"]) <= TOL[32]["vol"]
    assert abs(np.linalg.norm(x) / G["c3_per_inner_norm"][0] - 1) <= 1e-5


def test_radix5_side_320_vs_unmodified_reference(monkeypatch):
    """A common cryo-EM box with a factor 5 (320 = 2^6 * 5: radix-5 stages in
    every transform) through the C ABI the drop-in adapter calls, against the
    UNMODIFIED reference m_step run live (oracle/_ref): reference default
    semantics, 2 iterations, fp32 bar."""
    from oracle_lib import Reference, have_reference, make_cfg
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    monkeypatch.setenv("CM_REF_FFT_THREADS", "8")  # the reference's FFT backend threads only
    n = 320
    p = synth.synthetic_problem(n)
    R = Reference()
    rc, sy, sn = R.scale_data(p.weight, p.numerator)
    assert rc == 0
    rc, base = R.derive_config(sy, sn, p.eps, p.eps_prime)
    c = make_cfg(alpha=base.alpha, beta=base.beta, gamma=base.gamma, eps=base.eps,
                 eps_prime=base.eps_prime, mu=base.mu, inner_iters=2)
    rc, xr, trr = R.m_step(p.weight, p.numerator, p.x0, p.x0, c)
    assert rc == 0, R.last_error()
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx = cm.Context(n, 32)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    np.testing.assert_allclose([s.s_y, s.s_n], [sy, sn], rtol=1e-12)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 2
    trace = []
    ctx.set_volumes(p.x0, p.x0)
    ctx.solve(cfg, trace)
    x = ctx.get_volume()
    ctx.close()
    check_trace(trace, trr, TOL[32]["obj"])
    assert rel(x, xr) <= TOL[32]["vol"]
