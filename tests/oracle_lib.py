"""ctypes bindings for the two CPU oracles — TEST INFRASTRUCTURE.

* ``Oracle``    -> oracle/_ref/liboracle.so, the C restatement (oracle/cm_oracle.c)
* ``Reference`` -> oracle/_ref/libcryomap_ref.so, the unmodified reference library
                   (built from /root/reference sources by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
leg import this module. Both take and return numpy float64 / complex128
arrays in the reference's x-fastest layout ([k][j][i] in C order).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_DIR = ROOT / "oracle" / "_ref"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class RegConfigC(C.Structure):
    """Leading fields of cm_reg_config / or_reg_config / RegConfig."""

    _fields_ = [
        ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
        ("eps", C.c_double), ("eps_prime", C.c_double), ("mu", C.c_double),
        ("inner_iters", C.c_int), ("step_rule", C.c_int), ("fixed_step", C.c_double),
        ("refresh", C.c_int), ("convex_mode", C.c_int),
    ]


def make_cfg(**kw) -> RegConfigC:
    c = RegConfigC()
    c.alpha, c.beta, c.gamma = 0.0, 0.0, 0.0
    c.eps, c.eps_prime, c.mu = 1e-3, 1e-3, 1e-5
    c.inner_iters, c.step_rule, c.fixed_step, c.refresh, c.convex_mode = 24, 0, 0.0, 0, 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _d(a: np.ndarray):
    assert a.dtype in (np.float64, np.complex128) and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build_oracles() -> None:
    """(Re)build oracle/_ref via oracle/Makefile (reference parts only when
    /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8"], check=True)


class _Lib:
    prefix = ""
    libname = ""

    def __init__(self):
        path = REF_DIR / self.libname
        if not path.exists():
            build_oracles()
        self.lib = C.CDLL(str(path))

    def f(self, name):
        return getattr(self.lib, self.prefix + name)


class Oracle(_Lib):
    prefix = "or_"
    libname = "liboracle.so"

    def __init__(self):
        super().__init__()
        self.f("smoothed_tv_value").restype = C.c_double
        self.f("symmetry_residue").restype = C.c_double

    # --- numerics
    def discrete_gradient(self, x):
        x = np.ascontiguousarray(x, np.float64)
        d = [np.empty_like(x) for _ in range(3)]
        self.f("discrete_gradient")(x.shape[0], _d(x), _d(d[0]), _d(d[1]), _d(d[2]))
        return d

    def gradient_adjoint(self, d1, d2, d3):
        out = np.empty_like(d1)
        self.f("gradient_adjoint")(d1.shape[0], _d(d1), _d(d2), _d(d3), _d(out))
        return out

    def fft3(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.shape, np.complex128)
        self.f("fft3")(x.shape[0], _d(x), _d(out))
        return out

    def compute_weights(self, x, eps, eps_prime, convex=False):
        x = np.ascontiguousarray(x, np.float64)
        a, b = np.empty_like(x), np.empty_like(x)
        self.f("compute_weights")(x.shape[0], _d(x), C.c_double(eps), C.c_double(eps_prime),
                                  int(convex), _d(a), _d(b))
        return a, b

    def smoothed_tv_value(self, x, mu, w_tv=None):
        x = np.ascontiguousarray(x, np.float64)
        return self.f("smoothed_tv_value")(x.shape[0], _d(x), C.c_double(mu),
                                           None if w_tv is None else _d(w_tv))

    def smoothed_tv_gradient(self, x, mu, w_tv=None):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        self.f("smoothed_tv_gradient")(x.shape[0], _d(x), C.c_double(mu),
                                       None if w_tv is None else _d(w_tv), _d(out))
        return out

    def symmetry_residue(self, w, y):
        return self.f("symmetry_residue")(w.shape[0], _d(w), _d(y))

    def data_gradient(self, w, y, x, finalized=True):
        out = np.empty_like(x)
        rc = self.f("data_gradient")(x.shape[0], _d(w), _d(y), int(finalized), _d(x), _d(out))
        return rc, out

    def prox_l1(self, x, t):
        out = np.empty_like(x)
        self.f("prox_l1")(x.shape[0], _d(x), _d(t), _d(out))
        return out

    def penalized_objective(self, w, y, x, cfg, anchor, wsrc, finalized=True):
        out = np.zeros(7)
        rc = self.f("penalized_objective")(x.shape[0], _d(w), _d(y), int(finalized), _d(x),
                                           C.byref(cfg), _d(anchor), _d(wsrc), _d(out))
        return rc, out

    def m_step(self, w, y, x_init, x_anchor, cfg, trace=True, finalized=True):
        out = np.zeros_like(x_init)
        tr = np.zeros((max(cfg.inner_iters, 1), 15)) if trace else None
        rows = C.c_int(0)
        rc = self.f("m_step")(x_init.shape[0], _d(w), _d(y), int(finalized), _d(x_init),
                              _d(x_anchor), C.byref(cfg), _d(out),
                              None if tr is None else _d(tr), C.byref(rows))
        return rc, out, (tr[: rows.value] if tr is not None else None)

    def scale_data(self, w, y, finalized=True):
        a, b = C.c_double(), C.c_double()
        rc = self.f("scale_data")(w.shape[0], _d(w), _d(y), int(finalized), C.byref(a),
                                  C.byref(b))
        return rc, a.value, b.value

    def derive_config(self, s_y, s_n, eps, eps_prime, a=0.45, b=1.8, g=0.1):
        out = RegConfigC()
        rc = self.f("derive_config")(C.c_double(s_y), C.c_double(s_n), C.c_double(eps),
                                     C.c_double(eps_prime), C.c_double(a), C.c_double(b),
                                     C.c_double(g), C.byref(out))
        return rc, out


def _preload_mkl() -> None:
    """The reference's FFTW shim runs on oneMKL DFTI from libtorch_cpu.so
    (oracle/fftw_shim/fftw_shim_mkl.c). Load that library RTLD_GLOBAL before the
    reference: loaded after numpy's OpenBLAS without it, the process aborts at
    exit (free(): invalid pointer)."""
    import importlib.util

    spec = importlib.util.find_spec("torch")
    if spec and spec.origin:
        lib = Path(spec.origin).parent / "lib" / "libtorch_cpu.so"
        if lib.exists():
            C.CDLL(str(lib), mode=C.RTLD_GLOBAL)


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref/libcryomap_ref.so)."""

    prefix = "ref_"
    libname = "libcryomap_ref.so"

    def __init__(self):
        _preload_mkl()
        super().__init__()
        self.f("last_error").restype = C.c_char_p

    def last_error(self) -> str:
        return self.f("last_error")().decode()

    def m_step(self, w, y, x_init, x_anchor, cfg, trace=True, finalized=True):
        out = np.zeros_like(x_init)
        tr = np.zeros((max(cfg.inner_iters, 1), 15)) if trace else None
        rows, secs = C.c_int(0), C.c_double(0.0)
        rc = self.f("m_step")(x_init.shape[0], _d(w), _d(y), int(finalized), _d(x_init),
                              _d(x_anchor), C.byref(cfg), _d(out),
                              None if tr is None else _d(tr), C.byref(rows), C.byref(secs))
        self.last_seconds = secs.value
        return rc, out, (tr[: rows.value] if tr is not None else None)

    def data_gradient(self, w, y, x, finalized=True):
        out = np.empty_like(x)
        rc = self.f("data_gradient")(x.shape[0], _d(w), _d(y), int(finalized), _d(x), _d(out))
        return rc, out

    def penalized_objective(self, w, y, x, cfg, anchor, wsrc, finalized=True):
        out = np.zeros(7)
        rc = self.f("penalized_objective")(x.shape[0], _d(w), _d(y), int(finalized), _d(x),
                                           C.byref(cfg), _d(anchor), _d(wsrc), _d(out))
        return rc, out

    def compute_weights(self, x, eps, eps_prime, convex=False):
        a, b = np.empty_like(x), np.empty_like(x)
        rc = self.f("compute_weights")(x.shape[0], _d(x), C.c_double(eps),
                                       C.c_double(eps_prime), int(convex), _d(a), _d(b))
        assert rc == 0
        return a, b

    def smoothed_tv_value(self, x, mu, w_tv=None):
        out = C.c_double()
        self.f("smoothed_tv_value")(x.shape[0], _d(x), C.c_double(mu),
                                    None if w_tv is None else _d(w_tv), C.byref(out))
        return out.value

    def smoothed_tv_gradient(self, x, mu, w_tv=None):
        out = np.empty_like(x)
        self.f("smoothed_tv_gradient")(x.shape[0], _d(x), C.c_double(mu),
                                       None if w_tv is None else _d(w_tv), _d(out))
        return out

    def prox_l1(self, x, t):
        out = np.empty_like(x)
        self.f("prox_l1")(x.shape[0], _d(x), _d(t), _d(out))
        return out

    def discrete_gradient(self, x):
        d = [np.empty_like(x) for _ in range(3)]
        self.f("discrete_gradient")(x.shape[0], _d(x), _d(d[0]), _d(d[1]), _d(d[2]))
        return d

    def scale_data(self, w, y, finalized=True):
        a, b = C.c_double(), C.c_double()
        rc = self.f("scale_data")(w.shape[0], _d(w), _d(y), int(finalized), C.byref(a),
                                  C.byref(b))
        return rc, a.value, b.value

    def derive_config(self, s_y, s_n, eps, eps_prime, a=0.45, b=1.8, g=0.1):
        out = RegConfigC()
        rc = self.f("derive_config")(C.c_double(s_y), C.c_double(s_n), C.c_double(eps),
                                     C.c_double(eps_prime), C.c_double(a), C.c_double(b),
                                     C.c_double(g), C.byref(out))
        return rc, out

    def fft3(self, x):
        out = np.empty(x.shape, np.complex128)
        self.f("fft3")(x.shape[0], _d(x), _d(out))
        return out

    def fft3_centered(self, x):
        out = np.empty(x.shape, np.complex128)
        self.f("fft3_centered")(x.shape[0], _d(x), _d(out))
        return out

    def fsc_volumes(self, a, b):
        """fsc(fft3_centered(a), fft3_centered(b)) by the reference (fsc.cpp)."""
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(a.shape[0] // 2 + 1)
        rc = self.f("fsc_volumes")(a.shape[0], _d(a), _d(b), _d(out))
        assert rc == 0, self.last_error()
        return out

    def backproject(self, inp, threads=1):
        """backproject_accumulate (backproject.cpp:12) on a BackprojectInput
        -> (status, weight, numerator)."""
        n = inp.side_n
        w = np.zeros((n, n, n))
        y = np.zeros((n, n, n), np.complex128)
        p = lambda a: C.c_void_p(a.ctypes.data if a.size else None)  # noqa: E731
        rc = self.f("backproject")(
            n, inp.images.shape[0], p(inp.images), p(inp.image_params), inp.poses.shape[0],
            p(inp.poses), inp.shifts.shape[0], p(inp.shifts), C.c_longlong(inp.entry_posterior.size),
            p(inp.entry_particle), p(inp.entry_candidate), p(inp.entry_posterior),
            int(inp.kernel_kind), C.c_double(inp.bandwidth), C.c_double(inp.radius_cutoff),
            int(threads), _d(w), C.c_void_p(y.ctypes.data))
        return rc, w, y

    def estep(self, inp, volume, sigma2, prune_floor=1e-8, threads=1):
        """e_step (estep.cpp:64) -> (status, dense posterior [images][candidates])."""
        n = inp.side_n
        V = np.ascontiguousarray(volume, np.complex128)
        s2 = np.ascontiguousarray(sigma2, np.float64)
        out = np.zeros((inp.images.shape[0], inp.poses.shape[0] * inp.shifts.shape[0]))
        p = lambda a: C.c_void_p(a.ctypes.data if a.size else None)  # noqa: E731
        rc = self.f("estep")(
            n, inp.images.shape[0], p(inp.images), p(inp.image_params), inp.poses.shape[0],
            p(inp.poses), inp.shifts.shape[0], p(inp.shifts), int(inp.kernel_kind),
            C.c_double(inp.bandwidth), C.c_double(inp.radius_cutoff), s2.size, p(s2),
            C.c_double(prune_floor), p(V), int(threads), _d(out))
        return rc, out

    def write_mrc_volume(self, path, x, voxel_size=1.0):
        """write_mrc(path, Volume3D) by the reference (mrc.cpp:134)."""
        x = np.ascontiguousarray(x, np.float64)
        return self.f("write_mrc_volume")(os.fsencode(str(path)), x.shape[0],
                                          C.c_double(voxel_size), _d(x))

    def read_mrc_volume(self, path, n):
        """read_mrc_volume(path) by the reference -> (status, volume, voxel size)."""
        out = np.zeros((n, n, n))
        vs = C.c_double(0.0)
        rc = self.f("read_mrc_volume")(os.fsencode(str(path)), n, _d(out), C.byref(vs))
        return rc, out, vs.value

    def symmetry_residue(self, w, y):
        out = C.c_double()
        self.f("symmetry_residue")(w.shape[0], _d(w), _d(y), C.byref(out))
        return out.value

    def phantom(self, n, n_blobs, seed):
        out = np.zeros((n, n, n))
        rc = self.f("phantom")(n, n_blobs, C.c_ulonglong(seed), _d(out))
        assert rc == 0, self.last_error()
        return out


def have_reference() -> bool:
    return (REF_DIR / "libcryomap_ref.so").exists() or os.path.isdir("/root/reference/proj/src")
