"""GPU parity tests: the sm_100a solver (through the C ABI) against the
reference's golden vectors (tests/golden, produced by the unmodified
reference) and the oracle restatement on identical seeded inputs.

Tolerances (BASELINE.json north_star):
  fp32 (product mode): per-iteration objective fields within 1e-5 relative
                       (relative to max(|field|, |surrogate|)), final volume
                       within 1e-4 relative L2.
  fp64 (parity mode):  1e-9 relative — the reference's own audit slack.
"""
import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from golden.make_golden import CONFIGS, random_accumulator, random_volume, sha
from oracle_lib import Oracle, make_cfg

pytestmark = pytest.mark.gpu

G = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "reference_golden.npz")
TOL = {32: dict(obj=1e-5, vol=1e-4, pt=2e-5), 64: dict(obj=1e-9, vol=1e-9, pt=1e-10)}


@pytest.fixture(scope="module")
def O():
    return Oracle()


def acc_of(w, y, finalized=True):
    return cm.AccumulatorPair(w.shape[0], y, w, finalized)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check_trace(rows, ref, tol):
    got = np.array([np.r_[r.before.as_array(), r.after.as_array(), r.step] for r in rows])
    assert got.shape == ref.shape, (got.shape, ref.shape)
    for half in (slice(0, 7), slice(7, 14)):
        g, r = got[:, half], ref[:, half]
        surr = np.abs(r[:, 0] + r[:, 1] + r[:, 2] + r[:, 4])
        scale = np.maximum(np.abs(r), surr[:, None])
        err = np.abs(g - r) / scale
        assert err.max() <= tol, (half, err.max(), np.unravel_index(err.argmax(), err.shape))
    np.testing.assert_allclose(got[:, 14], ref[:, 14], rtol=1e-12)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n", [4, 6, 8, 10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 100,
                               112, 128, 160, 200, 224])
def test_fft3_matches_reference_convention(n, prec):
    """fourier.hpp:6-9: unnormalised forward transform (test_grid_fourier KATs)."""
    x = np.random.default_rng(n).standard_normal((n, n, n))
    F = cm.fft3(x, precision=prec)
    want = np.fft.fftn(x)
    tol = 1e-12 if prec == 64 else 2e-6
    assert np.abs(F - want).max() <= tol * np.abs(want).max()
    d = np.zeros((n, n, n))
    d[0, 0, 0] = 1.0
    np.testing.assert_allclose(cm.fft3(d, precision=prec), np.ones((n, n, n)), atol=tol)


def test_fft3_golden():
    x = random_volume(6, 3)
    np.testing.assert_allclose(cm.fft3(x, precision=64), G["fft6"], atol=1e-12)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n,seed", [(6, 11), (8, 12)])
def test_data_gradient_and_scales_golden(n, seed, prec):
    w, y = random_accumulator(n, seed)
    x = random_volume(n, seed + 100)
    assert sha(w, y, x) == str(G[f"racc{n}_sha"])
    acc = acc_of(w, y)
    g = cm.data_gradient(x, acc, precision=prec)
    ref = G[f"racc{n}_dgrad"]
    assert np.abs(g - ref).max() <= TOL[prec]["pt"] * max(1.0, np.abs(ref).max()) * 10
    s = cm.scale_data(acc, precision=prec)
    np.testing.assert_allclose([s.s_y, s.s_n], G[f"racc{n}_scales"], rtol=1e-12)
    ctx = cm.context(n, prec)
    assert abs(ctx.accumulator_info()[0] - G[f"racc{n}_resid"][0]) < 1e-15


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n", [16, 32])
def test_m_step_traces_golden(n, prec):
    """Per-iteration ObjectiveValue (before/after) and final volume of the
    reference m_step, four RegConfig modes."""
    p = synth.synthetic_problem(n)
    k = f"prob{n}"
    assert sha(p.weight, p.numerator, p.x0) == str(G[k + "_sha"])
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    np.testing.assert_allclose([s.s_y, s.s_n], G[k + "_scales"], rtol=1e-12)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    np.testing.assert_allclose([base.alpha, base.beta, base.gamma, base.eps, base.eps_prime,
                                base.mu], G[k + "_cfg"], rtol=1e-12)
    # x0 is the exact data-term minimiser (Y = W fft3_centered(x0)), so the
    # reference gradient is pure roundoff: compare on the scale of x0
    g = cm.data_gradient(p.x0, acc, precision=prec)
    ref = G[k + "_dgrad"]
    assert np.abs(g - ref).max() <= TOL[prec]["pt"] * np.abs(p.x0).max()
    for name, extra in CONFIGS.items():
        tr_ref = G[f"{k}_{name}_trace"]
        cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": len(tr_ref),
                              "fixed_step": float(G[f"{k}_{name}_fixed_step"][0])})
        for kk, vv in extra.items():
            setattr(cfg, kk, vv)
        trace = []
        x = cm.m_step(acc, p.x0, p.x0, cfg, trace, precision=prec)
        check_trace(trace, tr_ref, TOL[prec]["obj"])
        assert rel_l2(x, G[f"{k}_{name}_x"]) <= TOL[prec]["vol"], name


@pytest.mark.parametrize("prec", [32, 64])
def test_penalized_objective_golden(prec):
    n = 16
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    c = G["prob16_cfg"]
    cfg = cm.RegConfig(alpha=c[0], beta=c[1], gamma=c[2], eps=c[3], eps_prime=c[4], mu=c[5])
    xp = p.x0 + 0.05 * random_volume(n, 7)
    o = cm.penalized_objective(xp, acc, cfg, p.x0, p.x0, precision=prec).as_array()
    ref = G["prob16_obj"]
    assert np.max(np.abs(o - ref) / np.maximum(np.abs(ref), 1.0)) <= TOL[prec]["obj"]


@pytest.mark.parametrize("prec", [32, 64])
def test_components_vs_oracle(O, prec):
    n = 12
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n, n, n))
    w = rng.uniform(0.2, 3.0, (n, n, n))
    tol = TOL[prec]["pt"] * 10
    a, b = O.compute_weights(x, 0.01, 0.004)
    got = cm.compute_weights(x, 0.01, 0.004, precision=prec)
    np.testing.assert_allclose(got.w_l1, a, rtol=tol)
    np.testing.assert_allclose(got.w_tv, b, rtol=tol)
    for wt in (None, w):
        g = cm.smoothed_tv_gradient(x, 0.2, wt, precision=prec)
        ref = O.smoothed_tv_gradient(x, 0.2, wt)
        assert np.abs(g - ref).max() <= tol * np.abs(ref).max()
        v = cm.smoothed_tv_value(x, 0.2, wt, precision=prec)
        assert abs(v - O.smoothed_tv_value(x, 0.2, wt)) <= tol * abs(v)
    t = rng.uniform(0, 1, (n, n, n))
    np.testing.assert_array_equal(cm.prox_l1(x, t, precision=prec), O.prox_l1(x, t))


@pytest.mark.parametrize("prec", [32, 64])
def test_unregularized_convergence_and_l1_kill(prec):
    """test_regularizer.cpp:331-358."""
    n = 6
    w = synth.symmetric_weight(n, 21)
    target = random_volume(n, 22)
    acc = acc_of(w, w * synth.fft3_centered(target))
    z = np.zeros((n, n, n))
    x = cm.m_step(acc, z, z, cm.RegConfig(inner_iters=50), precision=prec)
    assert np.abs(x - target).max() < (1e-6 if prec == 64 else 1e-5)
    cfg = cm.RegConfig(alpha=1e12, beta=0.0, gamma=0.2, eps=0.05, eps_prime=0.02, mu=2e-4,
                       inner_iters=3)
    x = cm.m_step(acc, random_volume(n, 23), z, cfg, precision=prec)
    assert np.all(x == 0.0)


@pytest.mark.parametrize("prec", [32, 64])
def test_error_behaviour(prec):
    n = 6
    w = synth.symmetric_weight(n, 1)
    y = w * synth.fft3_centered(random_volume(n, 2))
    x = random_volume(n, 3)
    with pytest.raises(cm.NonHermitianAccumulator):
        cm.data_gradient(x, acc_of(w, y, finalized=False), precision=prec)
    yb = y.copy()
    yb[0, 0, 1] += 1.0
    with pytest.raises(cm.NonHermitianAccumulator):
        cm.m_step(acc_of(w, yb), x, x, cm.RegConfig(inner_iters=2), precision=prec)
    with pytest.raises(cm.InvalidArgument):
        cm.m_step(acc_of(w, y), x, x, cm.RegConfig(alpha=-1.0), precision=prec)
    with pytest.raises(cm.GridMismatch):
        cm.m_step(acc_of(w, y), np.zeros((8, 8, 8)), x, cm.RegConfig(), precision=prec)


@pytest.mark.parametrize("prec", [32, 64])
def test_config1_64cubed_vs_oracle(O, prec):
    """BASELINE config 1 at full size: 64^3, 100 iterations, one reweighting pass
    (per_m_step), lipschitz audit on, against the oracle restatement."""
    n = 64
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 100
    cfg.refresh = cm.Refresh.per_m_step
    trace = []
    x = cm.m_step(acc, p.x0, p.x0, cfg, trace, precision=prec)
    c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                 eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=100, refresh=1)
    rc, xo, tro = O.m_step(p.weight, p.numerator, p.x0, p.x0, c)
    assert rc == 0
    check_trace(trace, tro, TOL[prec]["obj"])
    assert rel_l2(x, xo) <= TOL[prec]["vol"]


SWEEP_MODES = {
    "per_inner": dict(),
    "per_m_step_anchor_differs": dict(refresh=1),
    "convex": dict(convex_mode=1),
    "fixed": dict(step_rule=1),
}


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n", [12, 20, 28, 48, 80, 96, 112, 128, 160])
def test_sweep_tiles_and_modes_vs_oracle(O, n, prec):
    """Tile geometries of the fused sweep (TJ x TK line tiles, i-chunks, idle
    FFT groups) in every RegConfig mode, anchor != x_init, against the oracle."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    anchor = p.x0 + 0.01 * random_volume(n, 99)
    lr0 = 1.0 / (2.0 * p.weight.max() + 2.0 * base.gamma + 12.0 * base.beta / base.eps_prime / base.mu)
    for name, extra in SWEEP_MODES.items():
        cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 8, "fixed_step": 2.0 * lr0, **extra})
        trace = []
        x = cm.m_step(acc, p.x0, anchor, cfg, trace, precision=prec)
        c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                     eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=8,
                     step_rule=int(cfg.step_rule), fixed_step=cfg.fixed_step,
                     refresh=int(cfg.refresh), convex_mode=int(cfg.convex_mode))
        rc, xo, tro = O.m_step(p.weight, p.numerator, p.x0, anchor, c)
        assert rc == 0
        check_trace(trace, tro, TOL[prec]["obj"])
        assert rel_l2(x, xo) <= TOL[prec]["vol"], name


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n", [20, 28, 40, 56])
def test_radix5_radix7_sides_vs_unmodified_reference(n, prec):
    """Sides with factors 5 and 7 (radix-5 / radix-7 stages of the FFT engine)
    against the UNMODIFIED reference m_step (oracle/_ref, FFTW-API shim):
    reference default semantics, 12 iterations, traces and volume."""
    from oracle_lib import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = Reference()
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    rc, sy, sn = R.scale_data(p.weight, p.numerator)
    assert rc == 0
    s = cm.scale_data(acc, precision=prec)
    np.testing.assert_allclose([s.s_y, s.s_n], [sy, sn], rtol=1e-12)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 12
    trace = []
    x = cm.m_step(acc, p.x0, p.x0, cfg, trace, precision=prec)
    c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                 eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=12)
    rc, xr, trr = R.m_step(p.weight, p.numerator, p.x0, p.x0, c)
    assert rc == 0, R.last_error()
    check_trace(trace, trr, TOL[prec]["obj"])
    assert rel_l2(x, xr) <= TOL[prec]["vol"]


@pytest.mark.parametrize("prec", [32, 64])
def test_fista_reaches_the_ista_fixed_point(prec):
    """FISTA (opt-in) is judged on the converged volume against a long ISTA run
    (frozen weights: a convex subproblem)."""
    n = 16
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    # a better-conditioned instance (smaller TV weight) so ISTA converges in budget
    base.beta *= 0.01
    ista = cm.RegConfig(**{**base.__dict__, "inner_iters": 20000, "refresh": cm.Refresh.per_m_step,
                           "step_rule": cm.StepRule.fixed})
    lr = 1.0 / (2.0 * p.weight.max() + 2.0 * base.gamma + 12.0 * base.beta / base.eps_prime / base.mu)
    ista.fixed_step = lr
    xi = cm.m_step(acc, p.x0, p.x0, ista, precision=prec)
    fista = cm.RegConfig(**{**ista.__dict__, "inner_iters": 3000, "momentum": 1})
    st = {}
    xf = cm.m_step(acc, p.x0, p.x0, fista, precision=prec, stats=st)
    assert st["iterations"] == 3000
    assert rel_l2(xf, xi) < 2e-4


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n", [16, 128])
def test_fista_restart_reaches_the_ista_fixed_point_faster(n, prec):
    """FISTA with gradient-based adaptive restart (momentum = 2) converges to
    the same fixed point as long ISTA, and reaches the step-norm rule in no
    more iterations than plain FISTA."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    base.beta *= 0.01
    ista = cm.RegConfig(**{**base.__dict__, "inner_iters": 20000, "refresh": cm.Refresh.per_m_step,
                           "step_rule": cm.StepRule.fixed})
    lr = 1.0 / (2.0 * p.weight.max() + 2.0 * base.gamma + 12.0 * base.beta / base.eps_prime / base.mu)
    ista.fixed_step = lr
    xi = cm.m_step(acc, p.x0, p.x0, ista, precision=prec)
    fr = cm.RegConfig(**{**ista.__dict__, "inner_iters": 3000, "momentum": 2})
    xr = cm.m_step(acc, p.x0, p.x0, fr, precision=prec)
    assert rel_l2(xr, xi) < 2e-4
    stops = {}
    for mom in (1, 2):
        c = cm.RegConfig(**{**ista.__dict__, "inner_iters": 20000, "momentum": mom, "tol_kind": 2,
                            "tol": 1e-3})
        st = {}
        cm.m_step(acc, p.x0, p.x0, c, precision=prec, stats=st)
        assert st["stop_reason"] == 2
        stops[mom] = st["iterations"]
    assert stops[2] <= stops[1], stops


def test_tolerance_stop_matches_oracle_trace(O):
    """tol_kind=1 stops at the first iteration whose frozen-weight surrogate
    decrease falls below tol; the returned volume is that iterate."""
    n = 16
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=64)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    c = make_cfg(alpha=base.alpha, beta=base.beta, gamma=base.gamma, eps=base.eps,
                 eps_prime=base.eps_prime, mu=base.mu, inner_iters=400, refresh=1)
    rc, xo, tro = O.m_step(p.weight, p.numerator, p.x0, p.x0, c)
    sb = tro[:, 0] + tro[:, 1] + tro[:, 2] + tro[:, 4]
    sa = tro[:, 7] + tro[:, 8] + tro[:, 9] + tro[:, 11]
    rel = np.abs(sb - sa) / np.abs(sb)
    tol = float(np.quantile(rel, 0.5))
    want = int(np.argmax(rel < tol))  # first trace row whose decrease is below tol
    cfg = cm.RegConfig(alpha=base.alpha, beta=base.beta, gamma=base.gamma, eps=base.eps,
                       eps_prime=base.eps_prime, mu=base.mu, inner_iters=400,
                       refresh=cm.Refresh.per_m_step, tol_kind=1, tol=tol)
    st = {}
    cm.m_step(acc, p.x0, p.x0, cfg, precision=64, stats=st)
    assert st["stop_reason"] == 2
    # row i compares x_i and x_{i+1}; the solve stops there and returns x_{i+1}
    assert st["iterations"] == want + 1


@pytest.mark.parametrize("n", [128, 256])
def test_vector_path_without_trace_matches_trace_run(n):
    """The fp32 4-voxel stencil path skips trace-only terms when no trace is
    requested; the iterates, the audit and the tolerance stop must not change."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=32)
    base = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 12})
    trace = []
    x_tr = cm.m_step(acc, p.x0, p.x0, cfg, trace, precision=32)
    x_nt = cm.m_step(acc, p.x0, p.x0, cfg, precision=32)
    np.testing.assert_array_equal(x_tr, x_nt)
    sb = np.array([r.before.surrogate() for r in trace])
    sa = np.array([r.after.surrogate() for r in trace])
    assert np.all(sa <= sb + 1e-6 * np.abs(sb))  # monotone frozen-weight surrogate
    rel = np.abs(sb - sa) / np.abs(sb)
    tol = float(np.sort(rel)[len(rel) // 2])
    want = int(np.argmax(rel < tol))
    st = {}
    cm.m_step(acc, p.x0, p.x0, cm.RegConfig(**{**cfg.__dict__, "tol_kind": 1, "tol": tol}),
              precision=32, stats=st)
    assert st["stop_reason"] == 2 and st["iterations"] == want + 1


@pytest.mark.parametrize("n", [256])
def test_fused_plane_pairs_match_separate_passes(n, monkeypatch):
    """The opt-in fused y/x plane-pair kernels (CM_FUSED=1, xyfused.cuh) give the
    same iterates and audit as the separate passes."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=32)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 10
    t_sep, t_fus = [], []
    x_sep = cm.m_step(acc, p.x0, p.x0, cfg, t_sep, precision=32)
    monkeypatch.setenv("CM_FUSED", "1")
    ctx = cm.Context(n, 32)   # the flag is read when a context is created
    ctx.set_accumulator(acc)
    ctx.set_volumes(p.x0, p.x0)
    st = ctx.solve(cfg, t_fus)
    x_fus = ctx.get_volume()
    assert st.kernel_launches < 8 * 10 + 2   # 6 kernels per iteration when fused
    assert rel_l2(x_fus, x_sep) <= 1e-6
    np.testing.assert_allclose([r.after.surrogate() for r in t_fus],
                               [r.after.surrogate() for r in t_sep], rtol=1e-6)


@pytest.mark.parametrize("n", [256, 512])
@pytest.mark.parametrize("mode", ["per_inner", "per_m_step", "fista"])
def test_fused_k1_cluster_kernel_matches_separate_passes(n, mode, monkeypatch):
    """The opt-in fused K1 (CM_K1F=1, k1f.cuh: x C2R + stencil + x R2C in one
    thread-block-cluster kernel over distributed shared memory) gives the same
    iterates and audit trace as the separate x-transform kernels."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=32)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 8
    if mode == "per_m_step":
        cfg.refresh = cm.Refresh.per_m_step
    if mode == "fista":
        cfg.refresh = cm.Refresh.per_m_step
        cfg.momentum = 1
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("CM_K1F", flag)
        ctx = cm.Context(n, 32)   # the flag is read when a context is created
        ctx.set_accumulator(acc)
        ctx.set_volumes(p.x0, p.x0)
        tr = []
        st = ctx.solve(cfg, tr)
        out[flag] = (ctx.get_volume(), tr, st)
        ctx.close()
    assert out["1"][2].kernel_launches < out["0"][2].kernel_launches  # two launches fewer
    assert rel_l2(out["1"][0], out["0"][0]) <= 1e-6
    np.testing.assert_allclose([r.after.surrogate() for r in out["1"][1]],
                               [r.after.surrogate() for r in out["0"][1]], rtol=1e-6)


@pytest.mark.parametrize("n", [256, 512])
@pytest.mark.parametrize("mode", ["per_inner", "fista_tol"])
def test_yzy_l2_pipeline_matches_separate_passes(n, mode, monkeypatch):
    """The opt-in y-forward + z + y-inverse L2 pipeline (CM_YZY=1, yzy.cuh: one
    persistent kernel, items claimed in order, per-group completion counters)
    gives the same iterates, audit trace and stop as the separate passes."""
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=32)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 9
    if mode == "fista_tol":  # early stop through the device flag inside a graph chunk
        cfg.refresh = cm.Refresh.per_m_step
        cfg.momentum = 1
        cfg.tol_kind = 2
        cfg.tol = 0.5
        cfg.inner_iters = 60
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("CM_YZY", flag)
        ctx = cm.Context(n, 32)
        ctx.set_accumulator(acc)
        ctx.set_volumes(p.x0, p.x0)
        tr = []
        st = ctx.solve(cfg, tr)
        out[flag] = (ctx.get_volume(), tr, st)
        ctx.close()
    assert out["1"][2].iterations == out["0"][2].iterations
    assert out["1"][2].stop_reason == out["0"][2].stop_reason
    assert rel_l2(out["1"][0], out["0"][0]) <= 1e-6
    np.testing.assert_allclose([r.after.surrogate() for r in out["1"][1]],
                               [r.after.surrogate() for r in out["0"][1]], rtol=1e-6)


@pytest.mark.parametrize("prec", [32, 64])
def test_config2_reweighting_loops_vs_oracle(O, prec):
    """BASELINE config 2 structure: bond-like (chain) phantom, three
    m_step calls with per_m_step reweighting, x_init <- previous output, anchor
    fixed at the initial volume (refine.cpp:181 pattern), against the oracle.
    128^3 and 6 inner iterations per loop keep the oracle within seconds; every
    loop starts both solvers from the oracle's previous output (per-call parity)
    and the GPU-only chain is checked at the end."""
    n, loops, iters = 128, 3, 6
    p = synth.synthetic_problem(n, kind="bonds")
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = iters
    cfg.refresh = cm.Refresh.per_m_step
    c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                 eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=iters, refresh=1)
    ctx = cm.Context(n, prec)
    ctx.set_accumulator(acc)
    x_ref, x_gpu = p.x0, p.x0
    for _ in range(loops):
        trace = []
        ctx.set_volumes(x_ref, p.x0)
        ctx.solve(cfg, trace)
        x_step = ctx.get_volume()
        rc, xo, tro = O.m_step(p.weight, p.numerator, x_ref, p.x0, c)
        assert rc == 0
        check_trace(trace, tro, TOL[prec]["obj"])
        assert rel_l2(x_step, xo) <= TOL[prec]["vol"]
        ctx.set_volumes(x_gpu, p.x0)
        ctx.solve(cfg)
        x_gpu = ctx.get_volume()
        x_ref = xo
    assert rel_l2(x_gpu, x_ref) <= 3 * TOL[prec]["vol"]


@pytest.mark.parametrize("prec", [32, 64])
def test_em_m_step_block_returns_centered_spectrum(prec):
    """refine.cpp:175-183: scale_data -> derive_config -> m_step -> V =
    fft3_centered(x), with V from the device (cm_get_spectrum) against numpy."""
    n = 64
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    x, V = cm.em_m_step(acc, p.x0, p.eps, p.eps_prime, inner_iters=6, precision=prec)
    s = cm.scale_data(acc, precision=prec)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 6
    np.testing.assert_array_equal(x, cm.m_step(acc, p.x0, p.x0, cfg, precision=prec))
    want = np.fft.fftn(synth.halfshift3(x))
    tol = 1e-12 if prec == 64 else 2e-6
    assert np.abs(V - want).max() <= tol * np.abs(want).max()


@pytest.mark.parametrize("prec", [32, 64])
def test_fsc_of_two_resident_half_maps_vs_reference(prec):
    """em_refine's FSC between the two half-map results (refine.cpp:194,
    fsc.cpp:10-42) computed on the device from two resident contexts, against the
    unmodified reference (fsc of fft3_centered volumes)."""
    from oracle_lib import Reference, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref not built")
    n = 48
    p = synth.synthetic_problem(n)
    acc = acc_of(p.weight, p.numerator)
    s = cm.scale_data(acc, precision=prec)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 4
    ctxs = []
    for x0 in (p.x0, p.x0 + 0.2 * random_volume(n, 5)):
        c = cm.Context(n, prec)
        c.set_accumulator(acc)
        c.set_volumes(x0, x0)
        c.solve(cfg)
        ctxs.append(c)
    got = ctxs[0].fsc(ctxs[1])
    want = Reference().fsc_volumes(ctxs[0].get_volume(), ctxs[1].get_volume())
    tol = 1e-12 if prec == 64 else 1e-5
    np.testing.assert_allclose(got, want, atol=tol, rtol=tol)
    assert got[0] > 0.99 and got.shape == (n // 2 + 1,)
