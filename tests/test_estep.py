"""Device E-step (cm_estep) against the unmodified reference e_step
(estep.cpp:64-270, through oracle/_ref) on identical inputs.

Bar: every posterior within 1e-10 (absolute; posteriors are in [0, 1]) and the
same set of surviving (nonzero) candidates per particle -- the pose pruning and
the prune_floor cut must agree. Device sums run in a different order and its
sin/cos/exp differ from glibc by an ulp, so agreement is to roundoff.
"""
import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from paper_1905_13408_b200.backproject import GAUSSIAN, TRILINEAR
from oracle_lib import Reference, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")


def problem(n, m, kind, cut, scale, seed, grid=True, r=1, n_poses=12):
    inp = synth.synthetic_backprojection(n, m, n_poses=n_poses, trans_radius=r, kernel_kind=kind,
                                         radius_cutoff=cut, seed=seed, grid_angles=grid)
    rng = np.random.default_rng(seed + 100)
    V = rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n))
    shells = np.arange(n // 2 + 1)
    sigma2 = scale * n * (1.0 + 0.05 * shells)
    return inp, V, sigma2


@needs_ref
def test_reference_wrapper_rows_normalised():
    R = Reference()
    inp, V, s2 = problem(8, 4, GAUSSIAN, -1.0, 1.0, 1)
    rc, post = R.estep(inp, V, s2)
    assert rc == 0, R.last_error()
    np.testing.assert_allclose(post.sum(axis=1), 1.0, rtol=1e-12)


CASES = [
    # n, images, kernel, cutoff, sigma scale, grid angles, shift radius
    (8, 6, GAUSSIAN, -1.0, 1.0, True, 1),
    (8, 6, TRILINEAR, -1.0, 1.0, False, 1),
    (16, 10, GAUSSIAN, 5.0, 0.5, True, 2),
    (16, 10, TRILINEAR, -1.0, 2.0, True, 1),
    (32, 8, GAUSSIAN, -1.0, 1.0, False, 2),
    (32, 8, GAUSSIAN, 10.0, 0.05, True, 1),  # peaked: pose pruning active
]


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n,m,kind,cut,scale,grid,r", CASES)
def test_matches_reference(n, m, kind, cut, scale, grid, r):
    R = Reference()
    inp, V, s2 = problem(n, m, kind, cut, scale, n + m, grid, r)
    rc, want = R.estep(inp, V, s2)
    assert rc == 0, R.last_error()
    ctx = cm.Context(n)
    got = cm.e_step(ctx, inp, s2, volume=V)
    ctx.close()
    np.testing.assert_array_equal(got != 0, want != 0)
    assert np.abs(got - want).max() <= 1e-10
    np.testing.assert_allclose(got.sum(axis=1), 1.0, rtol=1e-12)


# production-shaped grids: 128^2 images, >= 200 poses (odd: pass 2's tail group
# of one pose), the zero-shift-only grid (no pass-2 shifts), one CTA pair per pose
BIG_CASES = [
    # n, images, n_poses, shift radius, sigma scale, prune_floor
    (128, 24, 201, 2, 0.02, 1e-8),   # broad: ~2300 of 2613 candidates survive
    (128, 24, 201, 2, 0.005, 1e-8),  # peaked: pose pruning active, 6-75 survive
    (128, 16, 13, 0, 0.005, 1e-8),
    (64, 20, 211, 1, 0.003, 1e-6),   # 1-7 survivors, a larger floor
]


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n,m,npose,r,scale,floor", BIG_CASES)
def test_matches_reference_production_grids(n, m, npose, r, scale, floor):
    R = Reference()
    inp, V, s2 = problem(n, m, GAUSSIAN, -1.0, scale, 3 * n + m, True, r, n_poses=npose)
    rc, want = R.estep(inp, V, s2, prune_floor=floor, threads=8)
    assert rc == 0, R.last_error()
    ctx = cm.Context(n)
    got = cm.e_step(ctx, inp, s2, volume=V, prune_floor=floor)
    ctx.close()
    np.testing.assert_array_equal(got != 0, want != 0)
    assert np.abs(got - want).max() <= 1e-10
    np.testing.assert_allclose(got.sum(axis=1), 1.0, rtol=1e-12)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("batch_bytes", [None, "200000"])
def test_sparse_rows_match_reference_in_batches(monkeypatch, batch_bytes):
    """cm_estep_sparse: the PosteriorRow lists (ascending candidate order, as
    estep.cpp:257-263 pushes them) equal the reference's rows; a small
    CM_ESTEP_BATCH_BYTES forces many particle batches and a capacity retry."""
    if batch_bytes:
        monkeypatch.setenv("CM_ESTEP_BATCH_BYTES", batch_bytes)
    R = Reference()
    inp, V, s2 = problem(32, 23, GAUSSIAN, -1.0, 0.05, 41, True, 1, n_poses=37)
    rc, want = R.estep(inp, V, s2)
    assert rc == 0, R.last_error()
    ctx = cm.Context(32)
    row_ptr, cand, w = cm.e_step(ctx, inp, s2, volume=V, sparse=True)
    dense = cm.e_step(ctx, inp, s2, volume=V)
    ctx.close()
    assert row_ptr[0] == 0 and row_ptr[-1] == cand.size
    for i in range(want.shape[0]):
        c = cand[row_ptr[i]:row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
        np.testing.assert_array_equal(c, np.nonzero(want[i])[0])
        assert np.abs(w[row_ptr[i]:row_ptr[i + 1]] - want[i, c]).max() <= 1e-10
    np.testing.assert_array_equal(dense != 0, want != 0)
    ep, ec, ew = cm.sparse_entries(row_ptr, cand, w)
    dp, dc, dw = cm.posterior_entries(dense)
    np.testing.assert_array_equal(ep, dp)
    np.testing.assert_array_equal(ec, dc)


@pytest.mark.gpu
@needs_ref
def test_prune_floor_above_every_candidate_gives_empty_rows():
    """prune_floor larger than the best candidate's posterior: the reference
    pushes no entry (estep.cpp:257-263), the device writes zeros (not 0/0)."""
    R = Reference()
    inp, V, s2 = problem(16, 6, GAUSSIAN, -1.0, 1e6, 9, True, 1)  # flat posteriors
    rc, want = R.estep(inp, V, s2, prune_floor=0.9)
    assert rc == 0, R.last_error()
    ctx = cm.Context(16)
    got = cm.e_step(ctx, inp, s2, volume=V, prune_floor=0.9)
    ctx.close()
    assert np.isfinite(got).all()
    np.testing.assert_array_equal(got != 0, want != 0)
    assert np.abs(got - want).max() <= 1e-10
    assert (want.sum(axis=1) == 0).any()


@pytest.mark.gpu
@needs_ref
def test_spread_posteriors_exercise_many_candidates():
    """The parity cases above are not degenerate one-hot rows."""
    R = Reference()
    inp, V, s2 = problem(16, 10, GAUSSIAN, -1.0, 2.0, 26, True, 1)
    rc, want = R.estep(inp, V, s2)
    assert rc == 0
    assert (want > 0).sum(axis=1).max() > 3


@pytest.mark.gpu
def test_resident_volume_and_em_round():
    """V = fft3_centered of the resident solve result (volume=None) equals
    passing that spectrum from the host; then the posteriors feed the device
    backprojection and the next M-step with nothing but images on the host."""
    n = 16
    inp, _, s2 = problem(n, 8, GAUSSIAN, -1.0, 1.0, 5)
    p = synth.synthetic_problem(n)
    ctx = cm.Context(n, precision=64)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 4
    ctx.set_volumes(p.x0)
    ctx.solve(cfg)
    V = ctx.get_spectrum(centered=True)
    a = cm.e_step(ctx, inp, s2, volume=V)
    b = cm.e_step(ctx, inp, s2)
    np.testing.assert_array_equal(a != 0, b != 0)
    assert np.abs(a - b).max() <= 1e-12
    ep, ec, ew = cm.posterior_entries(b)
    inp.entry_particle, inp.entry_candidate, inp.entry_posterior = ep, ec, ew
    cm.backproject_into(ctx, inp, download=False)
    s2_ = ctx.scale_data()
    assert s2_.s_n > 0
    ctx.set_volumes(ctx.get_volume())
    ctx.solve(cfg)
    assert np.isfinite(ctx.get_volume()).all()
    ctx.close()


@pytest.mark.gpu
def test_errors():
    n = 8
    ctx = cm.Context(n)
    inp, V, s2 = problem(n, 2, GAUSSIAN, -1.0, 1.0, 3)
    no_zero = synth.synthetic_backprojection(n, 2, seed=3)
    no_zero.shifts = np.array([[1, 0]], np.int32)
    with pytest.raises(cm.InvalidArgument):
        cm.e_step(ctx, no_zero, s2, volume=V)
    empty = synth.synthetic_backprojection(n, 2, seed=3)
    empty.poses = np.zeros((0, 3))
    with pytest.raises(cm.InvalidArgument):
        cm.e_step(ctx, empty, s2, volume=V)
    with pytest.raises(cm.Error):  # no volume and no solver result resident
        cm.e_step(ctx, inp, s2)
    with pytest.raises(cm.GridMismatch):
        cm.e_step(ctx, inp, s2, volume=V[:4, :4, :4])
    ctx.close()


@pytest.mark.gpu
def test_resident_particles():
    """cm_set_particles once, then E-step and backprojection with images=NULL:
    the same posteriors (bitwise: the E-step has no atomics) and accumulator."""
    n = 16
    inp, V, s2 = problem(n, 8, GAUSSIAN, -1.0, 1.0, 8)
    ctx = cm.Context(n)
    with pytest.raises(cm.Error):  # nothing resident yet
        cm.e_step(ctx, inp, s2, volume=V, resident_images=True)
    cm.set_particles(ctx, inp)
    a = cm.e_step(ctx, inp, s2, volume=V)
    b = cm.e_step(ctx, inp, s2, volume=V, resident_images=True)
    np.testing.assert_array_equal(a, b)
    inp.entry_particle, inp.entry_candidate, inp.entry_posterior = cm.posterior_entries(b)
    x = cm.backproject_into(ctx, inp)
    y = cm.backproject_into(ctx, inp, resident_images=True)
    assert np.abs(x.numerator - y.numerator).max() <= 1e-13 * np.abs(x.numerator).max()
    assert np.abs(x.weight - y.weight).max() <= 1e-13 * x.weight.max()
    fewer = synth.synthetic_backprojection(n, 3, seed=1)
    with pytest.raises(cm.InvalidArgument):  # count differs from the resident set
        cm.e_step(ctx, fewer, s2, volume=V, resident_images=True)
    ctx.close()
