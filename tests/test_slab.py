"""z-slab decomposition.

CPU (gloo, world_size 2): the exchange pattern of csrc/dist.cuh — the
destination-major y-pass output, the all-to-all, the z transform on b rows,
the column-0 all-gather, the reverse transpose and the halo planes —
executed with numpy FFTs over torch.distributed, against the full-grid
transform. This pins SlabPlan's layout arithmetic (the same numbers the
device code uses) without a GPU.

GPU: the device z-slab solver with P ranks emulated on one B200 (exchanges
become device copies) against the single-GPU solver and the oracle.
"""
import os
import socket

import numpy as np
import pytest

import paper_1905_13408_b200 as cm
from paper_1905_13408_b200 import synth
from paper_1905_13408_b200.slab import SlabPlan


# ---------------------------------------------------------------------------------------
# host-side layout arithmetic
# ---------------------------------------------------------------------------------------
def test_plan_arithmetic():
    p = SlabPlan(512, 4)
    assert (p.nk, p.nb, p.nh) == (128, 128, 256)
    assert p.supported()
    assert not SlabPlan(256, 8).supported()      # 32 planes < one 64-plane march
    assert not SlabPlan(192, 1).supported()      # 128-wide stencil tiles
    assert list(p.planes(1)) == list(range(128, 256))
    g = p.ghosted_planes(0)
    assert g[0] is None and g[1] == 0 and g[-1] == 128
    assert p.ghosted_planes(3)[-1] is None
    assert p.halo_neighbours(0) == (None, 1) and p.halo_neighbours(3) == (2, None)
    # destination-major: chunk s (rows of rank s) is contiguous and chunk_elems long
    # destination-major with column halves: (half, peer) chunks are contiguous
    assert p.hh == 128 and p.chunk_elems() == 128 * 128 * 128
    assert p.dm_offset(0, 128, 0) == p.chunk_elems()
    assert p.dm_offset(p.nk - 1, p.nb - 1, p.hh - 1) == p.chunk_elems() - 1
    assert p.dm_offset(0, 0, p.hh) == p.half_elems() == 4 * p.chunk_elems()
    assert p.dm_offset(p.nk - 1, 511, p.nh - 1) == 2 * p.half_elems() - 1
    with pytest.raises(cm.InvalidArgument):
        SlabPlan(100, 3)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pack_half(F: np.ndarray, n: int) -> np.ndarray:
    """rfft over x (last axis) -> packed half spectrum: column 0 = X(0) + i X(n/2)."""
    S = F[..., : n // 2].copy()
    S[..., 0] = F[..., 0] + 1j * F[..., n // 2]
    return S


def _slab_worker(rank: int, world: int, port: int, n: int, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = SlabPlan(n, world)
        nk, nb, nh = plan.nk, plan.nb, plan.nh
        x = np.random.default_rng(7).standard_normal((n, n, n))   # [k][j][i]
        mine = x[plan.planes(rank)]
        # x R2C + y forward on my planes, written destination-major
        Fxy = np.fft.fft(np.fft.rfft(mine, axis=2), axis=1)        # [kl][b][a]
        S = _pack_half(Fxy, n)                                      # [kl][b][h]
        hh = plan.hh
        send = np.empty(2 * plan.half_elems(), np.complex128)
        for kl in range(nk):
            for b in range(n):
                for half in range(2):
                    o = plan.dm_offset(kl, b, half * hh)
                    send[o:o + hh] = S[kl, b, half * hh:(half + 1) * hh]
        # one all-to-all per column half: chunk s -> rank s
        sv = torch.from_numpy(send.view(np.float64).copy())
        rv = torch.empty_like(sv)
        he = 2 * plan.half_elems()  # float64 words per half
        for half in range(2):
            dist.all_to_all_single(rv[half * he:(half + 1) * he], sv[half * he:(half + 1) * he])
        halves = rv.numpy().view(np.complex128).reshape(2, world * nk, nb, hh)  # [half][c][bl][hh]
        recv = np.concatenate([halves[0], halves[1]], axis=2)                  # [c][bl][h]
        # z pass on my b rows
        Z = np.fft.fft(recv, axis=0)
        full = _pack_half(np.fft.fftn(x), n)                        # [c][b][h]
        ok_fwd = np.allclose(Z, full[:, plan.rows(rank), :], atol=1e-9 * n ** 3)
        # column 0 all-gather: every rank sees Z0[b][c] of the whole grid
        z0 = torch.from_numpy(np.ascontiguousarray(Z[:, :, 0].T).view(np.float64).copy())
        z0all = [torch.empty_like(z0) for _ in range(world)]
        dist.all_gather(z0all, z0)
        Z0 = np.concatenate([t.numpy().view(np.complex128) for t in z0all], axis=0)  # [b][c]
        ok_z0 = np.allclose(Z0, full[:, :, 0].T, atol=1e-9 * n ** 3)
        # Friedel pairing of the packed column: X(0) and X(n/2) planes per (b, c)
        b = plan.rows(rank)[0]
        c = np.arange(n)
        zz, zm = Z0[b, c], Z0[(-b) % n, (-c) % n]
        f0, fn = 0.5 * (zz + zm.conj()), (zz - zm.conj()) / 2j
        F = np.fft.fftn(x)
        ok_pair = np.allclose(f0, F[c, b, 0], atol=1e-9 * n ** 3) and \
            np.allclose(fn, F[c, b, n // 2], atol=1e-9 * n ** 3)
        # reverse transposes return my planes
        back = torch.empty_like(rv)
        for half in range(2):
            dist.all_to_all_single(back[half * he:(half + 1) * he], rv[half * he:(half + 1) * he])
        ok_back = np.array_equal(back.numpy(), sv.numpy())
        # halo: my last plane -> next rank's lower ghost, my first -> previous's upper
        lo_n, hi_n = plan.halo_neighbours(rank)
        ghost_lo = torch.zeros(n * n, dtype=torch.float64)
        ghost_hi = torch.zeros(n * n, dtype=torch.float64)
        reqs = []
        if hi_n is not None:
            reqs += [dist.isend(torch.from_numpy(mine[-1].ravel().copy()), hi_n),
                     dist.irecv(ghost_hi, hi_n)]
        if lo_n is not None:
            reqs += [dist.isend(torch.from_numpy(mine[0].ravel().copy()), lo_n),
                     dist.irecv(ghost_lo, lo_n)]
        for r in reqs:
            r.wait()
        g = plan.ghosted_planes(rank)
        ok_halo = True
        if g[0] is not None:
            ok_halo &= np.array_equal(ghost_lo.numpy(), x[g[0]].ravel())
        if g[-1] is not None:
            ok_halo &= np.array_equal(ghost_hi.numpy(), x[g[-1]].ravel())
        q.put((rank, bool(ok_fwd), bool(ok_z0), bool(ok_pair), bool(ok_back), bool(ok_halo)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [8, 12])
def test_slab_exchange_pattern_gloo(n):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert all(r[1:]), r


def _convert_rows(Wsrc, Ysrc, row_of, n, b):
    """dist.cuh convert_rows_kernel restated for one spectrum row b: the projected,
    sign-folded (W, Yh) over (c, a), a in [0, n/2], from accumulator rows held at
    row_of(b) and row_of(-b)."""
    c = np.arange(n)[:, None]
    a = np.arange(n // 2 + 1)[None, :]
    cm_, am, bm = (-c) % n, (-a) % n, (-b) % n
    w, wm = Wsrc[c, row_of(b), a], Wsrc[cm_, row_of(bm), am]
    y, ym = Ysrc[c, row_of(b), a], Ysrc[cm_, row_of(bm), am]
    sg = np.where((a + b + c) & 1, -1.0, 1.0)
    return 0.5 * (w + wm), sg * 0.5 * (y + ym.conj()), (w, wm, y, ym, a)


def _row_stats(parts, n):
    """acc_row_stats_kernel's five row terms (sum W, sum |Z_H|^2, max residue,
    max scale, max W)."""
    w, wm, y, ym, a = parts
    inner = (a != 0) & (a != n // 2)
    sw = np.where(inner, w + wm, w).sum()
    zh = 0.5 * (y / np.sqrt(w) + (ym / np.sqrt(wm)).conj())
    sz = (np.where(inner, 2.0, 1.0) * np.abs(zh) ** 2).sum()
    worst = max(np.abs(y - ym.conj()).max(), np.abs(w - wm).max())
    scale = max(np.abs(y).max(), w.max(), np.abs(ym).max(), wm.max())
    return np.array([sw, sz, worst, scale, max(w.max(), wm.max())])


def _acc_worker(rank: int, world: int, port: int, n: int, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = SlabPlan(n, world)
        rng = np.random.default_rng(11)
        W = rng.random((n, n, n)) + 0.5                                   # [c][b][a]
        Y = rng.standard_normal((n, n, n)) + 1j * rng.standard_normal((n, n, n))
        rows = plan.acc_rows(rank)
        local = {b: i for i, b in enumerate(rows)}
        Ws, Ys = W[:, rows, :], Y[:, rows, :]                              # what the rank uploads
        ok_conv, mine = True, []
        for b in plan.rows(rank):
            wp, yp, parts = _convert_rows(Ws, Ys, lambda r: local[r], n, b)  # KeyError: row missing
            wf, yf, _ = _convert_rows(W, Y, lambda r: r, n, b)
            ok_conv &= np.array_equal(wp, wf) and np.array_equal(yp, yf)
            mine.append(_row_stats(parts, n))
        mine = torch.from_numpy(np.array(mine).T.copy())                  # [5][nb]
        got = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(got, mine)
        allrows = torch.cat(got, dim=1).numpy()                          # [5][n], row order
        sw, sz = allrows[0].sum(), allrows[1].sum()                      # in row order
        one = np.array([_row_stats(_convert_rows(W, Y, lambda r: r, n, b)[2], n) for b in range(n)]).T
        ok_stats = (sw == one[0].sum() and sz == one[1].sum() and
                    allrows[2:].max(axis=1).tolist() == one[2:].max(axis=1).tolist())
        ok_bytes = (len(rows) <= min(n, 2 * plan.nb) and
                    plan.acc_upload_bytes(rank) == 24 * len(rows) * n * n)
        q.put((rank, bool(ok_conv), bool(ok_stats), bool(ok_bytes)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(8, 2), (16, 4)])
def test_sliced_accumulator_upload_gloo(n, world):
    """Each rank converts its b rows from only the accumulator rows it uploads
    (SlabPlan.acc_rows: its rows and their mirrors), bit-identical to converting
    from the full grid; the per-row statistics, all-gathered and summed in row
    order, equal the single-rank sums exactly."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_acc_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert all(r[1:]), r
    plan = SlabPlan(64, 8)
    assert plan.acc_rows(0) == [0] + list(range(1, 8)) + list(range(57, 64))
    assert plan.acc_rows(4) == list(range(25, 40))


# ---------------------------------------------------------------------------------------
# device solver, P ranks emulated on one GPU
# ---------------------------------------------------------------------------------------
MODES = {
    "per_inner": dict(),
    "per_m_step": dict(refresh=1),
    "convex": dict(convex_mode=1),
    "fixed": dict(step_rule=1),
}


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _traces(rows):
    return np.array([np.r_[r.before.as_array(), r.after.as_array(), r.step] for r in rows])


def _check_traces(a, b, tol, what=""):
    """Objective fields relative to max(|field|, |surrogate|) (test_gpu_parity.check_trace)."""
    assert a.shape == b.shape, what
    for half in (slice(0, 7), slice(7, 14)):
        surr = np.abs(b[:, half][:, [0, 1, 2, 4]].sum(axis=1))
        scale = np.maximum(np.abs(b[:, half]), surr[:, None])
        assert (np.abs(a[:, half] - b[:, half]) / scale).max() <= tol, what
    np.testing.assert_allclose(a[:, 14], b[:, 14], rtol=1e-12)


def _problem(n):
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    s = cm.scale_data(acc, precision=32)
    return p, acc, cm.derive_config(s.s_y, s.s_n, p.eps, p.eps_prime)


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(128, 2), (256, 2), (256, 4)])
def test_slab_matches_single_gpu(n, world):
    from paper_1905_13408_b200.slab import SlabContext

    p, acc, base = _problem(n)
    lr0 = 1.0 / (2.0 * p.weight.max() + 2.0 * base.gamma + 12.0 * base.beta / base.eps_prime / base.mu)
    sc = SlabContext(n, world)
    sc.set_accumulator(acc)
    sc.set_volumes(p.x0)
    for name, extra in MODES.items():
        cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 10, "fixed_step": 2.0 * lr0, **extra})
        t1, t2 = [], []
        x1 = cm.m_step(acc, p.x0, p.x0, cfg, t1, precision=32)
        sc.solve(cfg, t2)
        x2 = sc.get_volume()
        _check_traces(_traces(t2), _traces(t1), 1e-6, name)
        assert _rel(x2, x1) <= 1e-6, (name, _rel(x2, x1))
    sc.close()


@pytest.mark.gpu
def test_slab_sliced_upload_is_decomposition_independent():
    """Each emulated rank uploads only its accumulator rows (the bytes SlabPlan
    predicts, ~2/P of the full grid's); the volume is bit-identical to one rank's."""
    from paper_1905_13408_b200.slab import SlabContext

    n = 256
    p, acc, base = _problem(n)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 6})
    out = {}
    for world in (1, 4):
        sc = SlabContext(n, world)
        sc.set_accumulator(acc)
        plan = sc.plan
        assert sc.acc_upload_bytes == sum(plan.acc_upload_bytes(r) for r in range(world))
        sc.set_volumes(p.x0)
        t = []
        sc.solve(cfg, t)
        out[world] = (sc.get_volume(), _traces(t))
        sc.close()
    assert SlabPlan(n, 4).acc_upload_bytes(1) < 24 * n ** 3 // 2 + 1
    assert np.array_equal(out[4][0], out[1][0])
    # the objective partials are summed per rank, then across ranks: roundoff only
    np.testing.assert_allclose(out[4][1], out[1][1], rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_slab_vs_oracle_128():
    from oracle_lib import Oracle, make_cfg

    n = 128
    p, acc, base = _problem(n)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 8})
    trace = []
    x = cm.slab.m_step_slab(acc, p.x0, p.x0, cfg, world=2, trace=trace)
    c = make_cfg(alpha=cfg.alpha, beta=cfg.beta, gamma=cfg.gamma, eps=cfg.eps,
                 eps_prime=cfg.eps_prime, mu=cfg.mu, inner_iters=8)
    rc, xo, tro = Oracle().m_step(p.weight, p.numerator, p.x0, p.x0, c)
    assert rc == 0
    got = _traces(trace)
    surr = np.abs(tro[:, 0] + tro[:, 1] + tro[:, 2] + tro[:, 4])
    for half in (slice(0, 7), slice(7, 14)):
        err = np.abs(got[:, half] - tro[:, half]) / np.maximum(np.abs(tro[:, half]), surr[:, None])
        assert err.max() <= 1e-5
    assert _rel(x, xo) <= 1e-4


@pytest.mark.gpu
def test_slab_fista_tolerance_stop_matches_single_gpu():
    from paper_1905_13408_b200.slab import SlabContext

    n, world = 256, 4
    p, acc, base = _problem(n)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 400, "momentum": 1, "tol_kind": 2,
                          "tol": 0.05})
    st1 = {}
    x1 = cm.m_step(acc, p.x0, p.x0, cfg, precision=32, stats=st1)
    sc = SlabContext(n, world)
    sc.set_accumulator(acc)
    sc.set_volumes(p.x0)
    st2 = sc.solve(cfg)
    x2 = sc.get_volume()
    assert st1["stop_reason"] == 2 and st2.stop_reason == 2
    assert st2.iterations == st1["iterations"]
    assert _rel(x2, x1) <= 1e-6


@pytest.mark.gpu
def test_slab_errors():
    from paper_1905_13408_b200.slab import SlabContext

    with pytest.raises(cm.Error):
        SlabContext(192, 1)            # no 128-wide tiles
    with pytest.raises(cm.Error):
        SlabContext(256, 8)            # 32 planes per rank
    n = 128
    p, acc, base = _problem(n)
    sc = SlabContext(n, 2)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 2, "refresh": cm.Refresh.per_m_step})
    with pytest.raises(cm.Error):
        sc.solve(cfg)                  # accumulator not set
    sc.set_accumulator(acc)
    sc.set_volumes(p.x0, p.x0 + 1.0)   # anchor differs: frozen weights need x_init == anchor
    with pytest.raises(cm.Error):
        sc.solve(cfg)
    bad = cm.AccumulatorPair(n, p.numerator, p.weight, False)
    with pytest.raises(cm.NonHermitianAccumulator):
        sc.set_accumulator(bad)
        sc.solve(cm.RegConfig(**{**base.__dict__, "inner_iters": 2}))
    sc.close()


@pytest.mark.gpu
def test_slab_nccl_single_rank_matches_single_gpu():
    """The NCCL communicator (dlopen'd libnccl) at world size 1: init, all-gather,
    all-reduce on the solver stream."""
    from paper_1905_13408_b200.slab import SlabContext, nccl_unique_id

    n = 128
    p, acc, base = _problem(n)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 10})
    t1, t2 = [], []
    x1 = cm.m_step(acc, p.x0, p.x0, cfg, t1, precision=32)
    sc = SlabContext(n, 1, 0, 0, nccl_unique_id())
    sc.set_accumulator(acc)
    sc.set_volumes(p.x0)
    sc.solve(cfg, t2)
    x2 = sc.get_volume()
    sc.close()
    assert _rel(x2, x1) <= 1e-6
    _check_traces(_traces(t2), _traces(t1), 1e-6)  # partial sums regrouped per rank


@pytest.mark.gpu
def test_slab_nccl_all_to_all_path_single_rank(monkeypatch):
    """The grouped ncclSend/ncclRecv transposes (self send/recv at world size 1,
    CM_SLAB_FORCE_COMM) on the collectives stream: same solve as one GPU."""
    from paper_1905_13408_b200.slab import SlabContext, nccl_unique_id

    monkeypatch.setenv("CM_SLAB_FORCE_COMM", "1")
    n = 128
    p, acc, base = _problem(n)
    cfg = cm.RegConfig(**{**base.__dict__, "inner_iters": 8})
    x1 = cm.m_step(acc, p.x0, p.x0, cfg, precision=32)
    for nid in (nccl_unique_id(), None):   # NCCL, then the emulated communicator
        sc = SlabContext(n, 1, 0, 0, nid)
        sc.set_accumulator(acc)
        sc.set_volumes(p.x0)
        sc.solve(cfg)
        x2 = sc.get_volume()
        sc.close()
        assert _rel(x2, x1) <= 1e-6


@pytest.mark.gpu
def test_slab_synthetic_problem_is_decomposition_independent():
    """The device-rendered timing problem (bench 'big' runs) gives the same solve on
    1 and 4 ranks."""
    from paper_1905_13408_b200.slab import SlabContext

    n = 256
    out = []
    for world in (1, 4):
        sc = SlabContext(n, world)
        sy = sc.set_synthetic(7)
        cfg = cm.derive_config(sy, 1.5, 0.1, 0.1 / 3)
        cfg.inner_iters = 12
        st = sc.solve(cfg)
        assert st.stop_reason == 1 and st.iterations == 12
        out.append((sy, sc.get_volume()))
        sc.close()
    assert abs(out[0][0] - out[1][0]) <= 1e-12 * out[0][0]
    assert np.isfinite(out[0][1]).all()
    assert _rel(out[1][1], out[0][1]) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("ndev", [2, 4])
def test_multi_device_context_matches_one_gpu(ndev):
    """cm_ctx_create with ndev > 1 (the drop-in's multi-GPU path, CM_DEVICES in
    the C++ adapter): the z-slab runtime behind the ordinary cm_m_step /
    cm_scale_data entry points. With every device id equal the ranks are
    emulated on one GPU (the configuration a one-GPU box can run); the result
    and trace equal the one-GPU solver's."""
    import paper_1905_13408_b200 as cm
    from paper_1905_13408_b200 import synth
    n = 256
    p = synth.synthetic_problem(n)
    acc = cm.AccumulatorPair(n, p.numerator, p.weight, True)
    one = cm.Context(n, 32)
    one.set_accumulator(acc)
    s1 = one.scale_data()
    cfg = cm.derive_config(s1.s_y, s1.s_n, p.eps, p.eps_prime)
    cfg.inner_iters = 6
    out1 = np.empty((n, n, n))
    t1 = []
    one.set_volumes(p.x0, p.x0)
    one.solve(cfg, t1)
    out1 = one.get_volume()
    one.close()
    multi = cm.Context(n, 32, devices=[0] * ndev)
    multi.set_accumulator(acc)
    s2 = multi.scale_data()
    np.testing.assert_allclose([s2.s_y, s2.s_n], [s1.s_y, s1.s_n], rtol=1e-12)
    outm = np.empty((n, n, n))
    st = multi.m_step_host(acc, p.x0, p.x0, cfg, outm)
    multi.close()
    assert st.iterations == 6
    assert np.linalg.norm(outm - out1) / np.linalg.norm(out1) <= 1e-6


def test_multi_device_context_rejects_bad_layouts():
    """Host-side checks of cm_ctx_create(ndev > 1) (no device touched)."""
    import ctypes as C
    from paper_1905_13408_b200 import _lib
    lib = _lib.load()
    ptr = C.c_void_p()
    for n, devs, prec, why in [(256, [0, 1, 1], 32, "n / ndev"), (100, [0, 1], 32, "n % 128"),
                               (256, [0, 0], 64, "precision 32"),
                               (512, [0, 1, 1, 2], 32, "all distinct")]:
        arr = (C.c_int * len(devs))(*devs)
        assert lib.cm_ctx_create(n, arr, len(devs), prec, C.byref(ptr)) != 0
        assert why in lib.cm_last_error().decode(), (n, devs, lib.cm_last_error())
