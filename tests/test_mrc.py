"""MRC volume I/O on the resident volumes (cm_set_volumes_mrc /
cm_write_volume_mrc) against the reference's write_mrc / read_mrc_volume
(/root/reference/proj/src/mrc.cpp) run here through oracle/_ref.

Bar: byte-identical files from the writer; for the reader, the same status
(the reference's exception type) on every malformed file the reference's
reader rejects, and bit-identical solves from a file and from the same
volume rounded to float32 (mode 2) in memory.
"""
import struct

import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from oracle_lib import Reference, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")

OK, INVALID, GRID, IO, TRUNC, MAGIC, MODE = 0, 1, 2, 11, 12, 13, 14


def header(n, nz=None, mode=2, ispg=1, magic=b"MAP ", nsymbt=0):
    nz = n if nz is None else nz
    h = bytearray(1024)
    struct.pack_into("<3i", h, 0, n, n, nz)
    struct.pack_into("<i", h, 12, mode)
    struct.pack_into("<i", h, 88, ispg)
    struct.pack_into("<i", h, 92, nsymbt)
    struct.pack_into("<f", h, 40, float(n))
    h[208:212] = magic
    return bytes(h)


def malformed_files(tmp_path, n):
    """(name, bytes) pairs covering each rejection in read_mrc / read_mrc_volume."""
    pay = np.arange(n ** 3, dtype="<f4").tobytes()
    return {
        "short_header": b"\0" * 100,
        "bad_magic": header(n, magic=b"MAPX") + pay,
        "mode1": header(n, mode=1) + pay,
        "zero_dim": header(0) + pay,
        "neg_nsymbt": header(n, nsymbt=-4) + pay,
        "truncated": header(n) + pay[:-4],
        "stack": header(n, ispg=0) + pay,
        "nz_ne_nx": header(n, nz=n // 2) + pay,
        "side": header(n // 2) + pay,
    }


@needs_ref
def test_reference_reader_codes(tmp_path):
    """The crafted files hit the reference reader's own exception types."""
    R = Reference()
    want = {"short_header": TRUNC, "bad_magic": MAGIC, "mode1": MODE, "zero_dim": INVALID,
            "neg_nsymbt": INVALID, "truncated": TRUNC, "stack": INVALID, "nz_ne_nx": INVALID}
    n = 8
    for name, blob in malformed_files(tmp_path, n).items():
        if name not in want:
            continue
        f = tmp_path / f"{name}.mrc"
        f.write_bytes(blob)
        rc, _, _ = R.read_mrc_volume(f, n)
        assert rc == want[name], (name, rc, R.last_error())
    rc, _, _ = R.read_mrc_volume(tmp_path / "absent.mrc", n)
    assert rc == IO


@needs_ref
def test_reference_writer_layout(tmp_path):
    """The header fields the device writer reproduces (mrc.cpp:76-122)."""
    R = Reference()
    x = np.random.default_rng(3).standard_normal((8, 8, 8))
    f = tmp_path / "a.mrc"
    assert R.write_mrc_volume(f, x, 1.25) == OK
    b = f.read_bytes()
    assert len(b) == 1024 + 4 * 512
    assert struct.unpack_from("<4i", b, 0) == (8, 8, 8, 2)
    assert b[208:216] == b"MAP DD\0\0"
    np.testing.assert_array_equal(np.frombuffer(b, "<f4", offset=1024),
                                  x.astype(np.float32).ravel())


# ---------------------------------------------------------------------------- GPU
def solved_context(n, prec, iters=6):
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    s = cm.scale_data(acc, precision=prec)
    cfg = cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = iters
    ctx = cm.Context(n, precision=prec)
    ctx.set_accumulator(acc)
    return ctx, p, cfg


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("n,voxel", [(16, 1.0), (48, 1.37), (128, 0.83)])
def test_write_matches_reference_bytes(tmp_path, n, voxel, prec):
    R = Reference()
    ctx, p, cfg = solved_context(n, prec)
    ctx.set_volumes(p.x0)
    ctx.solve(cfg)
    ours, ref = tmp_path / "ours.mrc", tmp_path / "ref.mrc"
    ctx.write_volume_mrc(ours, voxel)
    assert R.write_mrc_volume(ref, ctx.get_volume(), voxel) == OK, R.last_error()
    assert ours.read_bytes() == ref.read_bytes()
    ctx.close()


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("prec", [32, 64])
def test_read_solves_like_the_float32_volume(tmp_path, prec):
    """A file written by the reference, loaded straight to the device, gives the
    solve the same volume gives after the reader's float32 -> double widening."""
    R = Reference()
    n = 32
    ctx, p, cfg = solved_context(n, prec)
    xi = p.x0 + 0.1 * np.random.default_rng(5).standard_normal(p.x0.shape)
    fi, fa = tmp_path / "init.mrc", tmp_path / "anchor.mrc"
    assert R.write_mrc_volume(fi, xi, 1.0) == OK
    assert R.write_mrc_volume(fa, p.x0, 1.0) == OK
    rc, xi_ref, _ = R.read_mrc_volume(fi, n)
    assert rc == OK
    _, xa_ref, _ = R.read_mrc_volume(fa, n)
    np.testing.assert_array_equal(xi_ref, xi.astype(np.float32).astype(np.float64))
    for anchor_path, anchor in ((None, xi_ref), (fa, xa_ref)):
        cfg.refresh = cm.Refresh.per_m_step
        ctx.set_volumes_mrc(fi, anchor_path)
        ctx.solve(cfg)
        from_file = ctx.get_volume()
        ctx.set_volumes(xi_ref, anchor)
        ctx.solve(cfg)
        np.testing.assert_array_equal(from_file, ctx.get_volume())
    ctx.close()


@pytest.mark.gpu
@needs_ref
def test_read_errors_match_reference(tmp_path):
    R = Reference()
    n = 8
    ctx, p, cfg = solved_context(n, 32)
    want_side = {"side": GRID}
    for name, blob in malformed_files(tmp_path, n).items():
        f = tmp_path / f"{name}.mrc"
        f.write_bytes(blob)
        rc = ctx.lib.cm_set_volumes_mrc(ctx.ptr, str(f).encode(), None)
        if name in want_side:
            assert rc == want_side[name], (name, rc)
            continue
        ref_rc, _, _ = R.read_mrc_volume(f, n)
        assert rc == ref_rc, (name, rc, ref_rc)
    rc = ctx.lib.cm_set_volumes_mrc(ctx.ptr, str(tmp_path / "absent.mrc").encode(), None)
    assert rc == IO
    with pytest.raises(OSError):
        ctx.set_volumes_mrc(tmp_path / "absent.mrc")
    # a file with an extended header is read past it (nsymbt, mrc.cpp:178)
    x = np.random.default_rng(1).standard_normal((n, n, n)).astype("<f4")
    f = tmp_path / "ext.mrc"
    f.write_bytes(header(n, nsymbt=96) + b"\x55" * 96 + x.tobytes())
    ctx.set_volumes_mrc(f)
    ctx.solve(cfg)
    a = ctx.get_volume()
    ctx.set_volumes(x.astype(np.float64))
    ctx.solve(cfg)
    np.testing.assert_array_equal(a, ctx.get_volume())
    # no result resident yet on a fresh context
    fresh = cm.Context(n, precision=32)
    assert fresh.lib.cm_write_volume_mrc(fresh.ptr, str(tmp_path / "o.mrc").encode(), 1.0) == 10
    fresh.close()
    ctx.close()


@pytest.mark.gpu
@needs_ref
def test_round_trip_at_512(tmp_path):
    """Production size: the 512^3 result written and read back through the
    pinned chunk ring (8 chunks) reproduces the reference writer's bytes."""
    R = Reference()
    n = 512
    ctx, p, cfg = solved_context(n, 32, iters=2)
    ctx.set_volumes(p.x0)
    ctx.solve(cfg)
    ours, ref = tmp_path / "ours.mrc", tmp_path / "ref.mrc"
    ctx.write_volume_mrc(ours, 1.1)
    x = ctx.get_volume()
    assert R.write_mrc_volume(ref, x, 1.1) == OK
    assert ours.read_bytes() == ref.read_bytes()
    ctx.set_volumes_mrc(ours)
    ctx.solve(cfg)
    a = ctx.get_volume()
    ctx.set_volumes(x)
    ctx.solve(cfg)
    np.testing.assert_array_equal(a, ctx.get_volume())
    ctx.close()
