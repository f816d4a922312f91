"""Python mirror of the reference solver interface, backed by the sm_100a library.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/cryomap/regularizer.hpp (RegConfig :21-35,
compute_weights :45-46, smoothed_tv_value/gradient :51-57, data_gradient :62,
prox_l1 :65, ObjectiveValue :67-79, penalized_objective :83-85,
MStepTraceRow :88-92, m_step :98-100), params.hpp (scale_data :22,
derive_config :39-41) and fourier.hpp (fft3 :11). Every call goes through the
C ABI in include/cm_api.h; there is no CPU fallback.

Volumes are numpy float64 arrays of shape (n, n, n) in the reference's
x-fastest layout (C order [k][j][i]); accumulators carry the full Fourier
grid (weight float64, numerator complex128), exactly like AccumulatorPair.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import cm_reg_config, cm_solve_stats, cm_trace_row


# ---- error types (errors.hpp:7-30) ------------------------------------------------
class Error(RuntimeError):
    pass


class InvalidArgument(Error):
    pass


class GridMismatch(Error):
    pass


class NonHermitianAccumulator(Error):
    pass


class StepDiverged(Error):
    pass


class NonPositiveScale(Error):
    pass


class NonHermitianInput(Error):
    pass


class DeviceError(Error):
    pass


_CODES = {
    1: InvalidArgument, 2: GridMismatch, 3: NonHermitianAccumulator, 4: StepDiverged,
    5: DeviceError, 6: DeviceError, 7: NonPositiveScale, 8: NonHermitianInput,
    9: InvalidArgument, 10: Error, 11: OSError, 12: OSError, 13: OSError, 14: OSError,
}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.load().cm_last_error().decode()
        raise _CODES.get(rc, Error)(msg)


# ---- configuration (regularizer.hpp:21-35) ----------------------------------------------
class StepRule(enum.IntEnum):
    lipschitz = 0
    fixed = 1


class Refresh(enum.IntEnum):
    per_inner = 0
    per_m_step = 1


@dataclass
class RegConfig:
    alpha: float = 0.0
    beta: float = 0.0
    gamma: float = 0.0
    eps: float = 1e-3
    eps_prime: float = 1e-3
    mu: float = 1e-5
    inner_iters: int = 24
    step_rule: StepRule = StepRule.lipschitz
    fixed_step: float = 0.0
    refresh: Refresh = Refresh.per_inner
    convex_mode: bool = False
    # extensions (defaults reproduce the reference)
    momentum: int = 0        # 1 = FISTA, 2 = FISTA with gradient adaptive restart
    tol_kind: int = 0        # 1 surrogate relative decrease, 2 step norm / max step
    tol: float = 0.0
    audit_slack: float = 0.0  # <= 0: 1e-9 (fp64) / 1e-6 (fp32)

    def to_c(self) -> cm_reg_config:
        c = cm_reg_config()
        c.alpha, c.beta, c.gamma = self.alpha, self.beta, self.gamma
        c.eps, c.eps_prime, c.mu = self.eps, self.eps_prime, self.mu
        c.inner_iters = int(self.inner_iters)
        c.step_rule = int(self.step_rule)
        c.fixed_step = self.fixed_step
        c.refresh = int(self.refresh)
        c.convex_mode = int(bool(self.convex_mode))
        c.momentum, c.tol_kind, c.tol = int(self.momentum), int(self.tol_kind), self.tol
        c.audit_slack = self.audit_slack
        return c


def validate_reg_config(config: RegConfig) -> None:
    """regularizer.cpp:33-42 (the library performs the same checks)."""
    if config.alpha < 0.0 or config.beta < 0.0 or config.gamma < 0.0:
        raise InvalidArgument("regularizer: alpha/beta/gamma must be >= 0")
    if config.eps <= 0.0 or config.eps_prime <= 0.0 or config.mu <= 0.0:
        raise InvalidArgument("regularizer: eps/eps_prime/mu must be > 0")
    if config.inner_iters < 1:
        raise InvalidArgument("regularizer: inner_iters must be >= 1")
    if config.step_rule == StepRule.fixed and config.fixed_step <= 0.0:
        raise InvalidArgument("regularizer: fixed step must be > 0")


@dataclass
class ObjectiveValue:
    fit: float = 0.0
    l1: float = 0.0
    tv_smooth: float = 0.0
    tv_linear: float = 0.0
    restraint: float = 0.0
    lognorm_l1: float = 0.0
    lognorm_tv: float = 0.0

    @classmethod
    def from_seq(cls, v) -> "ObjectiveValue":
        return cls(*[float(q) for q in v])

    def as_array(self) -> np.ndarray:
        return np.array([self.fit, self.l1, self.tv_smooth, self.tv_linear, self.restraint,
                         self.lognorm_l1, self.lognorm_tv])

    def surrogate(self) -> float:
        return self.fit + self.l1 + self.tv_smooth + self.restraint

    def surrogate_linear(self) -> float:
        return self.fit + self.l1 + self.tv_linear + self.restraint

    def lognorm(self) -> float:
        return self.fit + self.lognorm_l1 + self.lognorm_tv + self.restraint


@dataclass
class MStepTraceRow:
    before: ObjectiveValue
    after: ObjectiveValue
    step: float


@dataclass
class WeightFields:
    w_l1: np.ndarray
    w_tv: np.ndarray


@dataclass
class DataScales:
    s_y: float = 0.0
    s_n: float = 0.0


@dataclass
class Multipliers:
    a: float = 0.45
    b: float = 1.8
    g: float = 0.1


@dataclass
class AccumulatorPair:
    """backproject.hpp:15-25 — full Fourier grid, storage indices."""
    side_n: int
    numerator: np.ndarray  # complex128 (n, n, n)
    weight: np.ndarray     # float64 (n, n, n)
    finalized: bool = False
    voxel_size: float = 1.0


@dataclass
class SolveStats:
    iterations: int
    trace_rows: int
    stop_reason: int
    diverged_iter: int
    last_rel: float
    step: float
    solve_ms: float
    kernel_launches: int


def _arr(x):
    """Accept a numpy volume or a Volume3D-like object (side_n + data)."""
    return x.data if hasattr(x, "side_n") else x


# ---- context management ---------------------------------------------------------------------
def default_precision() -> int:
    return int(os.environ.get("CM_PRECISION", "32"))


class Context:
    """One cm_ctx: a side length, a precision, one GPU (or, with `devices`, the
    z-slab solver over several GPUs of the box; all ids equal: ranks emulated
    on that GPU); resident data in HBM."""

    def __init__(self, n: int, precision: int | None = None, device: int = 0,
                 devices: list[int] | None = None):
        lib = _lib.load()
        self.lib = lib
        self.n = int(n)
        self.precision = int(precision or default_precision())
        ptr = C.c_void_p()
        ids = list(devices) if devices else [device]
        dev = (C.c_int * len(ids))(*ids)
        _check(lib.cm_ctx_create(self.n, dev, len(ids), self.precision, C.byref(ptr)))
        self.ptr = ptr
        self._acc_key = None

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.lib.cm_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
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
        _check(self.lib.cm_set_accumulator(self.ptr, w.ctypes.data, y.ctypes.data,
                                           int(bool(acc.finalized))))

    def accumulator_info(self) -> tuple[float, float]:
        r, m = C.c_double(), C.c_double()
        _check(self.lib.cm_accumulator_info(self.ptr, C.byref(r), C.byref(m)))
        return r.value, m.value

    def set_volumes(self, x_init, x_anchor=None) -> None:
        xi = self._vol(x_init)
        if x_anchor is None or x_anchor is x_init:
            _check(self.lib.cm_set_volumes(self.ptr, xi.ctypes.data, xi.ctypes.data))
        else:
            xa = self._vol(x_anchor)
            _check(self.lib.cm_set_volumes(self.ptr, xi.ctypes.data, xa.ctypes.data))

    def solve(self, config: RegConfig, trace: list | None = None) -> SolveStats:
        cap = config.inner_iters if trace is not None else 0
        rows = (cm_trace_row * max(cap, 1))()
        st = cm_solve_stats()
        cfg = config.to_c()
        rc = self.lib.cm_solve(self.ptr, C.byref(cfg), rows if cap else None, cap, C.byref(st))
        if trace is not None:
            for r in range(st.trace_rows):
                trace.append(MStepTraceRow(ObjectiveValue.from_seq(rows[r].before),
                                           ObjectiveValue.from_seq(rows[r].after), rows[r].step))
        _check(rc)
        return SolveStats(st.iterations, st.trace_rows, st.stop_reason, st.diverged_iter,
                          st.last_rel, st.step, st.solve_ms, st.kernel_launches)

    def get_spectrum(self, centered: bool = True) -> np.ndarray:
        """fft3_centered (or fft3) of the resident solve result, complex128 (n, n, n):
        em_refine's V = fft3_centered(x) after m_step (refine.cpp:182), on the device."""
        out = np.empty((self.n,) * 3, dtype=np.complex128)
        _check(self.lib.cm_get_spectrum(self.ptr, int(bool(centered)), out.ctypes.data))
        return out

    def fsc(self, other: "Context") -> np.ndarray:
        """FSC curve (n/2 + 1 shells, fsc.cpp) between this context's resident result
        and another's (same device): em_refine's fsc(V_a, V_b), refine.cpp:194."""
        out = np.empty(self.n // 2 + 1, dtype=np.float64)
        _check(self.lib.cm_fsc(self.ptr, other.ptr, out.ctypes.data, out.size))
        return out

    def set_profiling(self, on: bool) -> None:
        _check(self.lib.cm_set_profiling(self.ptr, int(bool(on))))

    PROFILE_KERNELS = ("z_pass", "y_inverse", "x_c2r", "stencil", "finalize", "x_r2c", "y_forward")

    def get_profile(self) -> tuple[list[float], int]:
        """Accumulated per-kernel device ms (PROFILE_KERNELS order) and iterations."""
        ms = (C.c_double * 7)()
        it = C.c_int()
        _check(self.lib.cm_get_profile(self.ptr, ms, C.byref(it)))
        return list(ms), it.value

    def m_step_host(self, acc: AccumulatorPair, x_init, x_anchor, config: RegConfig,
                    out: np.ndarray | None = None) -> SolveStats:
        """One cm_m_step call on host buffers (upload, solve, download)."""
        w = np.ascontiguousarray(acc.weight, dtype=np.float64)
        y = np.ascontiguousarray(acc.numerator, dtype=np.complex128)
        xi = self._vol(x_init)
        xa = xi if (x_anchor is None or x_anchor is x_init) else self._vol(x_anchor)
        if out is None:
            out = np.empty((self.n,) * 3, np.float64)
        st = cm_solve_stats()
        cfg = config.to_c()
        _check(self.lib.cm_m_step(self.ptr, w.ctypes.data, y.ctypes.data, int(bool(acc.finalized)),
                                  xi.ctypes.data, xa.ctypes.data, C.byref(cfg), out.ctypes.data,
                                  None, 0, C.byref(st)))
        return SolveStats(st.iterations, st.trace_rows, st.stop_reason, st.diverged_iter,
                          st.last_rel, st.step, st.solve_ms, st.kernel_launches)

    def get_volume(self) -> np.ndarray:
        out = np.empty((self.n,) * 3, np.float64)
        _check(self.lib.cm_get_volume(self.ptr, out.ctypes.data))
        return out

    def set_volumes_mrc(self, path_init, path_anchor=None) -> None:
        """x_init (and x_anchor; None: the same object) from MRC files, read
        into pinned chunks and copied straight to the device (mrc.cpp:156
        checks and errors; cm_set_volumes_mrc)."""
        pa = None if path_anchor is None else os.fsencode(path_anchor)
        _check(self.lib.cm_set_volumes_mrc(self.ptr, os.fsencode(path_init), pa))

    def write_volume_mrc(self, path, voxel_size: float = 1.0) -> None:
        """The resident solve result as write_mrc(path, Volume3D(x, voxel_size))
        writes it, byte for byte (mrc.cpp:134; cm_write_volume_mrc)."""
        _check(self.lib.cm_write_volume_mrc(self.ptr, os.fsencode(path), float(voxel_size)))

    def scale_data(self) -> DataScales:
        a, b = C.c_double(), C.c_double()
        _check(self.lib.cm_scale_data(self.ptr, C.byref(a), C.byref(b)))
        return DataScales(a.value, b.value)


_tls = threading.local()


def context(n: int, precision: int | None = None, device: int = 0) -> Context:
    """Per-thread cached context (one per side / precision / device)."""
    key = (int(n), int(precision or default_precision()), device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if key not in cache:
        cache[key] = Context(*key)
    return cache[key]


def release_contexts() -> None:
    """Free this thread's cached contexts (their device memory)."""
    cache = getattr(_tls, "ctx", None)
    if cache:
        for c in cache.values():
            c.close()
        cache.clear()


def _side(x) -> int:
    return int(np.shape(_arr(x))[0])


# ---- reference API -------------------------------------------------------------------------
def m_step(acc: AccumulatorPair, x_init, x_anchor, config: RegConfig,
           trace: list | None = None, precision: int | None = None,
           stats: dict | None = None) -> np.ndarray:
    """regularizer.hpp:98-100 — inner_iters proximal-gradient iterations."""
    validate_reg_config(config)
    ctx = context(acc.side_n, precision)
    if _side(x_init) != acc.side_n or _side(x_anchor) != acc.side_n:
        raise GridMismatch("m_step: side_n differs")
    ctx.set_accumulator(acc)
    ctx.set_volumes(x_init, x_anchor)
    st = ctx.solve(config, trace)
    if stats is not None:
        stats.update(st.__dict__)
    return ctx.get_volume()


def em_m_step(acc: AccumulatorPair, x, eps: float, eps_prime: float,
              mult: Multipliers | None = None, inner_iters: int = 24,
              refresh: Refresh = Refresh.per_inner, convex_mode: bool = False,
              precision: int | None = None, extra: dict | None = None):
    """em_refine's regularized M-step block (refine.cpp:175-183) on one resident
    context: scale_data -> derive_config -> m_step(acc, x, x) -> V =
    fft3_centered(x). Returns (x_new, V); `extra` sets RegConfig extensions
    (momentum, tol_kind, tol). The data scales and V are computed on the device
    (no host FFT; the reference does two full-grid FFTs here per half-map)."""
    ctx = context(acc.side_n, precision)
    ctx.set_accumulator(acc)
    s = ctx.scale_data()
    cfg = derive_config(s.s_y, s.s_n, eps, eps_prime, mult)
    cfg.inner_iters = inner_iters
    cfg.refresh = refresh
    cfg.convex_mode = convex_mode
    for k, v in (extra or {}).items():
        setattr(cfg, k, v)
    ctx.set_volumes(x, x)
    ctx.solve(cfg)
    return ctx.get_volume(), ctx.get_spectrum(centered=True)


def data_gradient(x, acc: AccumulatorPair, precision: int | None = None) -> np.ndarray:
    """regularizer.hpp:62 — Re ifft3_centered(W .* fft3_centered(x) - num)."""
    if _side(x) != acc.side_n:
        raise GridMismatch("data_gradient: side_n differs")
    ctx = context(acc.side_n, precision)
    ctx.set_accumulator(acc)
    xa = ctx._vol(x)
    out = np.empty_like(xa)
    _check(ctx.lib.cm_data_gradient(ctx.ptr, xa.ctypes.data, out.ctypes.data))
    return out


def compute_weights(x_prev, eps: float, eps_prime: float, convex_mode: bool = False,
                    precision: int | None = None) -> WeightFields:
    ctx = context(_side(x_prev), precision)
    xa = ctx._vol(x_prev)
    a, b = np.empty_like(xa), np.empty_like(xa)
    _check(ctx.lib.cm_compute_weights(ctx.ptr, xa.ctypes.data, eps, eps_prime, int(convex_mode),
                                      a.ctypes.data, b.ctypes.data))
    return WeightFields(a, b)


def smoothed_tv_value(v, mu: float, w_tv=None, precision: int | None = None) -> float:
    ctx = context(_side(v), precision)
    xa = ctx._vol(v)
    w = None if w_tv is None else ctx._vol(w_tv)
    out = C.c_double()
    _check(ctx.lib.cm_smoothed_tv_value(ctx.ptr, xa.ctypes.data, mu,
                                        None if w is None else w.ctypes.data, C.byref(out)))
    return out.value


def smoothed_tv_gradient(v, mu: float, w_tv=None, precision: int | None = None) -> np.ndarray:
    ctx = context(_side(v), precision)
    xa = ctx._vol(v)
    w = None if w_tv is None else ctx._vol(w_tv)
    out = np.empty_like(xa)
    _check(ctx.lib.cm_smoothed_tv_gradient(ctx.ptr, xa.ctypes.data, mu,
                                           None if w is None else w.ctypes.data, out.ctypes.data))
    return out


def prox_l1(x_dash, thresholds, precision: int | None = None) -> np.ndarray:
    ctx = context(_side(x_dash), precision)
    xa = ctx._vol(x_dash)
    t = ctx._vol(thresholds)
    out = np.empty_like(xa)
    _check(ctx.lib.cm_prox_l1(ctx.ptr, xa.ctypes.data, t.ctypes.data, out.ctypes.data))
    return out


def penalized_objective(x, acc: AccumulatorPair, config: RegConfig, x_anchor,
                        x_weights_source, precision: int | None = None) -> ObjectiveValue:
    validate_reg_config(config)
    ctx = context(acc.side_n, precision)
    ctx.set_accumulator(acc)
    out = np.zeros(7)
    xs = [ctx._vol(q) for q in (x, x_anchor, x_weights_source)]
    cfg = config.to_c()
    _check(ctx.lib.cm_penalized_objective(ctx.ptr, xs[0].ctypes.data, C.byref(cfg),
                                          xs[1].ctypes.data, xs[2].ctypes.data, out.ctypes.data))
    return ObjectiveValue.from_seq(out)


def scale_data(acc: AccumulatorPair, precision: int | None = None) -> DataScales:
    """params.cpp:9-26."""
    if not acc.finalized:
        raise NonHermitianAccumulator("scale_data: accumulator is not finalized")
    ctx = context(acc.side_n, precision)
    ctx.set_accumulator(acc)
    return ctx.scale_data()


def derive_config(s_y: float, s_n: float, eps: float, eps_prime: float,
                  mult: Multipliers | None = None, warnings: list | None = None) -> RegConfig:
    """params.cpp:40-64."""
    mult = mult or Multipliers()
    lib = _lib.load()
    out = cm_reg_config()
    _check(lib.cm_derive_config(s_y, s_n, eps, eps_prime, mult.a, mult.b, mult.g, C.byref(out)))
    if warnings is not None:
        for name, v, lo, hi in (("alpha", mult.a, 0.4, 0.5), ("beta", mult.b, 1.2, 2.6),
                                ("gamma", mult.g, 0.05, 0.2)):
            if not (lo <= v <= hi):
                warnings.append(f"{name} multiplier {v:f} outside recommended [{lo:f}, {hi:f}]")
    return RegConfig(alpha=out.alpha, beta=out.beta, gamma=out.gamma, eps=out.eps,
                     eps_prime=out.eps_prime, mu=out.mu)


def fft3(v, precision: int | None = None) -> np.ndarray:
    """fourier.hpp:11 — unnormalised forward transform, full complex grid."""
    ctx = context(_side(v), precision)
    xa = ctx._vol(v)
    out = np.empty(xa.shape, np.complex128)
    _check(ctx.lib.cm_fft3(ctx.ptr, xa.ctypes.data, out.ctypes.data))
    return out


def fft3_centered(v, precision: int | None = None) -> np.ndarray:
    """fourier.hpp:24 (fourier.cpp:109) — fft3 of halfshift3(v), full complex grid."""
    ctx = context(_side(v), precision)
    xa = ctx._vol(v)
    out = np.empty(xa.shape, np.complex128)
    _check(ctx.lib.cm_fft3_centered(ctx.ptr, xa.ctypes.data, out.ctypes.data))
    return out
