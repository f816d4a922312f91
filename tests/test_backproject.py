"""Device backprojection (cm_backproject) against the unmodified reference
backproject_accumulate (backproject.cpp:12-101, run here through oracle/_ref).

Bar (the reference's own, test_em_engine.cpp:278-283): every numerator and
weight entry within 1e-10 of the largest magnitude; we hold 1e-12. The device
sums with fp64 atomics in no fixed order and its sin/cos/exp differ from glibc
by an ulp, so agreement is to roundoff, not bitwise. Friedel symmetry after
finalize is exact (test_em_engine.cpp:300-318).
"""
import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from paper_1905_13408_b200.backproject import GAUSSIAN, TRILINEAR
from oracle_lib import Reference, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
TOL = 1e-12


def mate(a):
    """a[mate(c), mate(b), mate(a)] in storage indices."""
    return np.roll(a[::-1, ::-1, ::-1], 1, axis=(0, 1, 2))


@needs_ref
def test_reference_wrapper_finalizes(tmp_path):
    R = Reference()
    inp = synth.synthetic_backprojection(8, 3, seed=1)
    rc, w, y = R.backproject(inp)
    assert rc == 0, R.last_error()
    assert np.abs(w).max() > 0
    np.testing.assert_array_equal(y, np.conj(mate(y)))
    np.testing.assert_array_equal(w, mate(w))


CASES = [
    # n, images, kernel, cutoff, grid angles, identity ctf, trans radius
    (6, 3, GAUSSIAN, -1.0, False, False, 1),
    (6, 3, TRILINEAR, -1.0, False, True, 1),
    (8, 5, GAUSSIAN, -1.0, True, False, 1),
    (8, 5, TRILINEAR, -1.0, True, False, 1),
    (16, 12, GAUSSIAN, 5.0, True, False, 2),
    (16, 12, TRILINEAR, 6.4, False, False, 2),
    (32, 20, GAUSSIAN, -1.0, True, False, 1),
    (32, 20, TRILINEAR, -1.0, True, True, 0),
    (48, 8, GAUSSIAN, 20.0, False, False, 1),
]


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("direct", ["0", "1"])
@pytest.mark.parametrize("n,m,kind,cut,grid,ident,r", CASES)
def test_matches_reference(n, m, kind, cut, grid, ident, r, direct, monkeypatch):
    """Both device forms: pose-grouped (default) and per-entry (CM_BP_DIRECT=1)."""
    monkeypatch.setenv("CM_BP_DIRECT", direct)
    R = Reference()
    inp = synth.synthetic_backprojection(n, m, n_poses=10, trans_radius=r, entries_per_image=4,
                                         kernel_kind=kind, radius_cutoff=cut, seed=n + m,
                                         grid_angles=grid, identity_ctf=ident)
    rc, w_ref, y_ref = R.backproject(inp)
    assert rc == 0, R.last_error()
    acc = cm.backproject_accumulate(inp)
    assert acc.finalized
    ys, ws = np.abs(y_ref).max(), w_ref.max()
    assert ys > 0 and ws > 0
    assert np.abs(acc.numerator - y_ref).max() <= TOL * ys
    assert np.abs(acc.weight - w_ref).max() <= TOL * ws
    # the zero pattern (which voxels any tap reached) is identical
    np.testing.assert_array_equal(acc.weight == 0, w_ref == 0)
    # exactly Friedel symmetric
    np.testing.assert_array_equal(acc.numerator, np.conj(mate(acc.numerator)))
    np.testing.assert_array_equal(acc.weight, mate(acc.weight))


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [32, 64])
def test_resident_accumulator_feeds_the_solver(prec):
    """backproject_into leaves the accumulator resident: the M-step after it is
    bit-identical to one after cm_set_accumulator of the same arrays."""
    n = 32
    inp = synth.synthetic_backprojection(n, 24, n_poses=16, entries_per_image=5, seed=3)
    ctx = cm.Context(n, precision=prec)
    acc = cm.backproject_into(ctx, inp, download=True)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, 1e-3, 1e-3)
    cfg.inner_iters = 8
    x0 = np.random.default_rng(0).standard_normal((n, n, n)) * 0.01
    ctx.set_volumes(x0)
    ctx.solve(cfg)
    a = ctx.get_volume()
    ctx.set_accumulator(acc)
    s2 = ctx.scale_data()
    assert (s2.s_y, s2.s_n) == (s.s_y, s.s_n)
    ctx.set_volumes(x0)
    ctx.solve(cfg)
    np.testing.assert_array_equal(a, ctx.get_volume())
    # no-download form gives the same resident state (to atomic-order roundoff)
    assert cm.backproject_into(ctx, inp, download=False) is None
    s3 = ctx.scale_data()
    np.testing.assert_allclose([s3.s_y, s3.s_n], [s.s_y, s.s_n], rtol=1e-13)
    ctx.close()


@pytest.mark.gpu
def test_errors_and_empty_rows():
    n = 8
    ctx = cm.Context(n, precision=32)
    inp = synth.synthetic_backprojection(n, 2, seed=4)
    bad = synth.synthetic_backprojection(n, 2, seed=4)
    bad.bandwidth = 0.0
    with pytest.raises(cm.InvalidArgument):
        cm.backproject_into(ctx, bad)
    bad = synth.synthetic_backprojection(n, 2, seed=4)
    bad.entry_particle[0] = 7
    with pytest.raises(cm.InvalidArgument):
        cm.backproject_into(ctx, bad)
    bad = synth.synthetic_backprojection(n, 2, seed=4)
    bad.entry_candidate[0] = 10 ** 6
    with pytest.raises(cm.InvalidArgument):
        cm.backproject_into(ctx, bad)
    with pytest.raises(cm.GridMismatch):
        cm.backproject_into(ctx, synth.synthetic_backprojection(6, 2, seed=4))
    # a failed call leaves no accumulator behind
    with pytest.raises(cm.Error):
        ctx.scale_data()
    # no entries (or only zero posteriors): a zero, finalized accumulator
    inp.entry_posterior[:] = 0.0
    acc = cm.backproject_into(ctx, inp)
    assert acc.finalized and not acc.weight.any() and not acc.numerator.any()
    ctx.close()


@pytest.mark.gpu
@needs_ref
def test_production_size_vs_reference_threads():
    """128^3 grid, 64 images x 4 candidates, Gaussian window: against the
    reference run with 8 worker threads (its deterministic merge)."""
    R = Reference()
    n = 128
    inp = synth.synthetic_backprojection(n, 64, n_poses=40, entries_per_image=4, seed=9)
    rc, w_ref, y_ref = R.backproject(inp, threads=8)
    assert rc == 0
    acc = cm.backproject_accumulate(inp)
    assert np.abs(acc.numerator - y_ref).max() <= TOL * np.abs(y_ref).max()
    assert np.abs(acc.weight - w_ref).max() <= TOL * w_ref.max()
