"""z-slab distributed M-step over the C ABI (cm_dctx_*).

One process per GPU. Rank r of P owns real-space planes k in [r NK, (r+1) NK)
(NK = n/P) with one ghost plane per side, and the spectrum rows b in
[r NB, (r+1) NB) (NB = n/P) for the z pass. Per iteration (csrc/dist.cuh):

    z pass on b rows -> all-gather of the packed column-0 pencils
    all-to-all (b-slab -> z-slab) -> y inverse -> x C2R -> stencil -> halo
    finalize (local partials -> all-reduce) -> x R2C -> y forward
    all-to-all (z-slab -> b-slab)

The y passes write the all-to-all send layout directly ([half][s][k][b_local][h],
``SlabPlan.dm_offset``), so the transposes need no packing kernels; the two
column halves are transposed separately, overlapping the other half's
transforms (collectives on their own stream).

``SlabPlan`` is the host-side arithmetic of that decomposition (the same
numbers dist.cuh uses); ``SlabContext`` drives the device solver. With
``nccl_id=None`` a SlabContext hosts all P ranks on one GPU (exchanges become
device copies) — that is how the decomposition is tested on a single B200.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import cm_reg_config, cm_solve_stats, cm_trace_row  # noqa: F401
from .regularizer import (AccumulatorPair, GridMismatch, InvalidArgument, MStepTraceRow,
                          ObjectiveValue, RegConfig, SolveStats, _arr, _check)


@dataclass(frozen=True)
class SlabPlan:
    """Decomposition of an n^3 grid over `world` ranks (dist.cuh DistImpl)."""

    n: int
    world: int

    def __post_init__(self):
        n, p = self.n, self.world
        if p < 1 or n % p:
            raise InvalidArgument(f"world {p} does not divide n {n}")

    @property
    def nk(self) -> int:  # real-space planes per rank
        return self.n // self.world

    @property
    def nb(self) -> int:  # spectrum rows per rank in the z pass
        return self.n // self.world

    @property
    def nh(self) -> int:
        return self.n // 2

    def supported(self) -> bool:
        """The device solver's constraint: 128-wide stencil tiles, 64-plane marches."""
        return self.n % 128 == 0 and self.nk % 64 == 0

    def planes(self, rank: int) -> range:
        return range(rank * self.nk, (rank + 1) * self.nk)

    def rows(self, rank: int) -> range:
        return range(rank * self.nb, (rank + 1) * self.nb)

    def acc_rows(self, rank: int) -> list[int]:
        """Accumulator rows b (of the full grid's [c][b][a]) that rank's b-slab
        conversion reads: its rows and their Friedel mirrors (n - b) mod n, sorted
        (csrc/dist.cuh acc_rows_needed; the rank uploads only these)."""
        need = set()
        for b in self.rows(rank):
            need.add(b)
            need.add((self.n - b) % self.n)
        return sorted(need)

    def acc_upload_bytes(self, rank: int) -> int:
        """fp64 W (8 B) + numerator (16 B) over the rank's accumulator rows."""
        return 24 * len(self.acc_rows(rank)) * self.n * self.n

    def ghosted_planes(self, rank: int) -> list[int | None]:
        """Global plane behind each local plane of the ghosted layout (None: outside)."""
        out = []
        for kl in range(-1, self.nk + 1):
            k = rank * self.nk + kl
            out.append(k if 0 <= k < self.n else None)
        return out

    @property
    def hh(self) -> int:  # columns per half: the spectrum's h range is split in two
        return self.nh // 2

    def half_elems(self) -> int:
        """Complex elements of one column half of a rank's spectrum block."""
        return self.nk * self.n * self.hh

    # destination-major spectrum layout with split column halves
    # [half][s][k_local][b_local][h - half hh] (kernels.cuh SpecLayout)
    def dm_offset(self, k_local: int, b: int, h: int) -> int:
        s, bl = divmod(b, self.nb)
        half, hl = divmod(h, self.hh)
        return half * self.half_elems() + ((s * self.nk + k_local) * self.nb + bl) * self.hh + hl

    def chunk_elems(self) -> int:
        """Complex elements each rank sends to each other rank per half transpose."""
        return self.nk * self.nb * self.hh

    def halo_neighbours(self, rank: int) -> tuple[int | None, int | None]:
        lo = rank - 1 if rank > 0 else None
        hi = rank + 1 if rank + 1 < self.world else None
        return lo, hi

    def exchange_bytes_per_iteration(self) -> int:
        """Bytes each rank sends per iteration (fp32): two transposes of two column
        halves, the column-0 all-gather, two halo planes and the partial-sum
        all-reduce."""
        p = self.world
        a2a = 2 * 2 * (p - 1) * self.chunk_elems() * 8
        z0 = (p - 1) * self.nb * self.n * 8
        halo = 2 * self.n * self.n * 4
        return a2a + z0 + halo + 13 * 8


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    buf = (C.c_ubyte * 128)()
    _check(lib.cm_nccl_unique_id(buf))
    return bytes(buf)


class SlabContext:
    """One cm_dctx: this process's ranks of a z-slab solve (fp32)."""

    def __init__(self, n: int, world: int, rank: int = 0, device: int = 0,
                 nccl_id: bytes | None = None):
        lib = _lib.load()
        self.lib = lib
        self.plan = SlabPlan(int(n), int(world))
        self.n = int(n)
        ptr = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise InvalidArgument("nccl_id must be 128 bytes")
            idbuf = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        _check(lib.cm_dctx_create(self.n, self.plan.world, int(rank), int(device), idbuf,
                                  C.byref(ptr)))
        self.ptr = ptr
        nk, first, here = C.c_int(), C.c_int(), C.c_int()
        _check(lib.cm_dctx_layout(ptr, C.byref(nk), C.byref(first), C.byref(here)))
        self.first_plane, self.ranks_here = first.value, here.value

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.lib.cm_dctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def local_planes(self) -> range:
        return range(self.first_plane, self.first_plane + self.ranks_here * self.plan.nk)

    def _vol(self, x) -> np.ndarray:
        a = np.ascontiguousarray(_arr(x), dtype=np.float64)
        if a.shape != (self.n,) * 3:
            raise GridMismatch(f"volume shape {a.shape} does not match side {self.n}")
        return a

    def set_accumulator(self, acc: AccumulatorPair) -> None:
        if acc.side_n != self.n:
            raise GridMismatch("accumulator side_n differs")
        w = np.ascontiguousarray(acc.weight, dtype=np.float64)
        y = np.ascontiguousarray(acc.numerator, dtype=np.complex128)
        if w.shape != (self.n,) * 3 or y.shape != (self.n,) * 3:
            raise GridMismatch("accumulator arrays do not match side_n")
        _check(self.lib.cm_dctx_set_accumulator(self.ptr, w.ctypes.data, y.ctypes.data,
                                                int(bool(acc.finalized))))

    @property
    def acc_upload_bytes(self) -> int:
        """Host-to-device bytes of this process's last set_accumulator."""
        v = C.c_longlong()
        _check(self.lib.cm_dctx_upload_bytes(self.ptr, C.byref(v)))
        return v.value

    def set_volumes(self, x_init, x_anchor=None) -> None:
        xi = self._vol(x_init)
        xa = xi if (x_anchor is None or x_anchor is x_init) else self._vol(x_anchor)
        _check(self.lib.cm_dctx_set_volumes(self.ptr, xi.ctypes.data, xa.ctypes.data))

    def solve(self, config: RegConfig, trace: list | None = None) -> SolveStats:
        cap = config.inner_iters if trace is not None else 0
        rows = (cm_trace_row * max(cap, 1))()
        st = cm_solve_stats()
        cfg = config.to_c()
        rc = self.lib.cm_dctx_solve(self.ptr, C.byref(cfg), rows if cap else None, cap,
                                    C.byref(st))
        if trace is not None:
            for r in range(st.trace_rows):
                trace.append(MStepTraceRow(ObjectiveValue.from_seq(rows[r].before),
                                           ObjectiveValue.from_seq(rows[r].after), rows[r].step))
        _check(rc)
        return SolveStats(st.iterations, st.trace_rows, st.stop_reason, st.diverged_iter,
                          st.last_rel, st.step, st.solve_ms, st.kernel_launches)

    def set_synthetic(self, seed: int = 1) -> float:
        """Device-rendered timing problem (no host accumulator); returns the volume RMS."""
        sy = C.c_double()
        _check(self.lib.cm_dctx_set_synthetic(self.ptr, C.c_ulonglong(seed), C.byref(sy)))
        return sy.value

    def get_volume(self, out: np.ndarray | None = None) -> np.ndarray:
        """Full-size array with this process's planes filled (others untouched)."""
        if out is None:
            out = np.zeros((self.n,) * 3, dtype=np.float64)
        if out.shape != (self.n,) * 3 or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise InvalidArgument("out must be a C-contiguous float64 (n, n, n) array")
        _check(self.lib.cm_dctx_get_volume(self.ptr, out.ctypes.data))
        return out


def m_step_slab(acc: AccumulatorPair, x_init, x_anchor, config: RegConfig,
                world: int, trace: list | None = None) -> np.ndarray:
    """m_step on `world` emulated z-slab ranks of the current GPU (decomposition check)."""
    ctx = SlabContext(acc.side_n, world)
    try:
        ctx.set_accumulator(acc)
        ctx.set_volumes(x_init, x_anchor)
        ctx.solve(config, trace)
        return ctx.get_volume()
    finally:
        ctx.close()
