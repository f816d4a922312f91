"""Device backprojection: backproject_accumulate (backproject.hpp:26-30,
backproject.cpp:12-101) through cm_backproject, SURVEY §8(f) rank 2.

The inputs are the reference's ParticleSet, PosteriorRow list and
OrientationGrid in flat arrays (include/cm_api.h, cm_bp_input). The
accumulator is produced on the device, Friedel-finalized, and left resident in
the context as its M-step accumulator; the host copy is optional.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .regularizer import AccumulatorPair, Context, _check


class cm_bp_input(C.Structure):
    _fields_ = [
        ("n_images", C.c_int),
        ("images", C.c_void_p),
        ("image_params", C.c_void_p),
        ("n_poses", C.c_int),
        ("poses", C.c_void_p),
        ("n_shifts", C.c_int),
        ("shifts", C.c_void_p),
        ("n_entries", C.c_longlong),
        ("entry_particle", C.c_void_p),
        ("entry_candidate", C.c_void_p),
        ("entry_posterior", C.c_void_p),
        ("kernel_kind", C.c_int),
        ("bandwidth", C.c_double),
        ("radius_cutoff", C.c_double),
    ]


GAUSSIAN, TRILINEAR = 0, 1  # KernelKind order, kernel.hpp:6


@dataclass
class BackprojectInput:
    """ParticleSet + posterior rows + OrientationGrid, flattened.

    images:          complex128 (m, n, n), ParticleImage::f (row l, column k,
                     storage indices)
    image_params:    float64 (m, 6): voltage_kv, defocus_A, cs_mm,
                     amplitude_contrast, identity_flag, voxel_size
    poses:           float64 (p, 3): rot, tilt, psi in degrees
    shifts:          int32 (s, 2): dx, dy
    entry_particle / entry_candidate / entry_posterior: one per (row, entry),
                     candidate = pose * s + shift (orientation.hpp:19-21)
    """
    images: np.ndarray
    image_params: np.ndarray
    poses: np.ndarray
    shifts: np.ndarray
    entry_particle: np.ndarray
    entry_candidate: np.ndarray
    entry_posterior: np.ndarray
    kernel_kind: int = GAUSSIAN
    bandwidth: float = 2.0
    radius_cutoff: float = -1.0

    def __post_init__(self):
        self.images = np.ascontiguousarray(self.images, np.complex128)
        self.image_params = np.ascontiguousarray(self.image_params, np.float64).reshape(-1, 6)
        self.poses = np.ascontiguousarray(self.poses, np.float64).reshape(-1, 3)
        self.shifts = np.ascontiguousarray(self.shifts, np.int32).reshape(-1, 2)
        self.entry_particle = np.ascontiguousarray(self.entry_particle, np.int64)
        self.entry_candidate = np.ascontiguousarray(self.entry_candidate, np.uint32)
        self.entry_posterior = np.ascontiguousarray(self.entry_posterior, np.float64)

    @property
    def side_n(self) -> int:
        return int(self.images.shape[-1])

    def to_c(self, resident_images: bool = False) -> cm_bp_input:
        d = lambda a: a.ctypes.data if a.size else None  # noqa: E731
        img = None if resident_images else d(self.images)
        par = None if resident_images else d(self.image_params)
        return cm_bp_input(
            int(self.images.shape[0]), img, par,
            int(self.poses.shape[0]), d(self.poses), int(self.shifts.shape[0]), d(self.shifts),
            int(self.entry_posterior.size), d(self.entry_particle), d(self.entry_candidate),
            d(self.entry_posterior), int(self.kernel_kind), float(self.bandwidth),
            float(self.radius_cutoff))


def set_particles(ctx: Context, inp: BackprojectInput) -> None:
    """Upload the particle images once (cm_set_particles); later calls with
    resident_images=True read them on the device."""
    d = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    _check(ctx.lib.cm_set_particles(ctx.ptr, int(inp.images.shape[0]), d(inp.images),
                                    d(inp.image_params)))


def backproject_into(ctx: Context, inp: BackprojectInput, download: bool = True,
                     resident_images: bool = False):
    """Accumulate on the device into ctx's resident accumulator (finalized);
    returns the AccumulatorPair copy when `download`."""
    n = ctx.n
    if inp.side_n != n:
        from .regularizer import GridMismatch
        raise GridMismatch(f"backproject: images of side {inp.side_n}, context side {n}")
    c = inp.to_c(resident_images)
    w = np.empty((n, n, n), np.float64) if download else None
    y = np.empty((n, n, n), np.complex128) if download else None
    _check(ctx.lib.cm_backproject(ctx.ptr, C.byref(c), None if w is None else w.ctypes.data,
                                  None if y is None else y.ctypes.data))
    if not download:
        return None
    vox = float(inp.image_params[0, 5]) if inp.image_params.size else 1.0
    return AccumulatorPair(n, y, w, True, vox)


def backproject_accumulate(inp: BackprojectInput, precision: int | None = None) -> AccumulatorPair:
    """backproject_accumulate (backproject.hpp:26) on the device, host result."""
    ctx = Context(inp.side_n, precision=precision)
    try:
        return backproject_into(ctx, inp, download=True)
    finally:
        ctx.close()


class cm_estep_input(C.Structure):
    _fields_ = [
        ("n_images", C.c_int),
        ("images", C.c_void_p),
        ("image_params", C.c_void_p),
        ("n_poses", C.c_int),
        ("poses", C.c_void_p),
        ("n_shifts", C.c_int),
        ("shifts", C.c_void_p),
        ("kernel_kind", C.c_int),
        ("bandwidth", C.c_double),
        ("radius_cutoff", C.c_double),
        ("n_sigma2", C.c_int),
        ("sigma2", C.c_void_p),
        ("prune_floor", C.c_double),
        ("volume", C.c_void_p),
    ]


def e_step(ctx: Context, inp: BackprojectInput, sigma2, volume=None,
           prune_floor: float = 1e-8, resident_images: bool = False, sparse: bool = False):
    """e_step (estep.hpp:44-54) on the device -> dense posterior
    [images][poses * shifts] (PosteriorRow entries at their candidate index,
    exact zeros elsewhere), or with sparse=True the PosteriorRow lists as
    (row_ptr [images+1], candidate, weight) (cm_estep_sparse: never dense).
    The particles, grid and kernel come from `inp` (its entry arrays are
    ignored); volume None: V = fft3_centered of ctx's resident solve result,
    never leaving the device."""
    n = ctx.n
    if inp.side_n != n:
        from .regularizer import GridMismatch
        raise GridMismatch(f"e_step: images of side {inp.side_n}, context side {n}")
    s2 = np.ascontiguousarray(sigma2, np.float64).ravel()
    V = None if volume is None else np.ascontiguousarray(volume, np.complex128)
    if V is not None and V.shape != (n, n, n):
        from .regularizer import GridMismatch
        raise GridMismatch("e_step: volume side differs from the context")
    d = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
    img = None if resident_images else d(inp.images)
    par = None if resident_images else d(inp.image_params)
    c = cm_estep_input(int(inp.images.shape[0]), img, par,
                       int(inp.poses.shape[0]), d(inp.poses), int(inp.shifts.shape[0]),
                       d(inp.shifts), int(inp.kernel_kind), float(inp.bandwidth),
                       float(inp.radius_cutoff), int(s2.size), d(s2), float(prune_floor), d(V))
    m = int(inp.images.shape[0])
    if sparse:
        row_ptr = np.zeros(m + 1, np.int64)
        cap = max(1, m * min(64, inp.poses.shape[0] * inp.shifts.shape[0]))
        while True:
            cand = np.empty(cap, np.int32)
            w = np.empty(cap, np.float64)
            nnz = C.c_longlong(0)
            rc = ctx.lib.cm_estep_sparse(ctx.ptr, C.byref(c), row_ptr.ctypes.data, cand.ctypes.data,
                                         w.ctypes.data, cap, C.byref(nnz))
            if rc != 0 and nnz.value > cap:  # capacity too small: the call says how many
                cap = int(nnz.value)
                continue
            _check(rc)
            return row_ptr, cand[: nnz.value].copy(), w[: nnz.value].copy()
    out = np.zeros((m, inp.poses.shape[0] * inp.shifts.shape[0]))
    _check(ctx.lib.cm_estep(ctx.ptr, C.byref(c), out.ctypes.data))
    return out


def sparse_entries(row_ptr, cand, weight):
    """cm_estep_sparse's PosteriorRow lists -> the flat (particle, candidate,
    weight) entry arrays of cm_bp_input."""
    part = np.repeat(np.arange(row_ptr.size - 1, dtype=np.int64), np.diff(row_ptr))
    return part, cand.astype(np.uint32), weight


def posterior_entries(dense: np.ndarray):
    """Dense posterior -> the flat (particle, candidate, weight) entry arrays
    of cm_bp_input, in PosteriorRow order."""
    part, cand = np.nonzero(dense)
    return part.astype(np.int64), cand.astype(np.uint32), dense[part, cand]
