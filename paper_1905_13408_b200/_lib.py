"""ctypes binding of libcm.so (include/cm_api.h). Fails loudly: there is no
CPU fallback anywhere in the product path."""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
HEADER = ROOT / "include" / "cm_api.h"
LIBPATH = Path(os.environ.get("CM_LIBRARY", str(PKG / "libcm.so")))

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class cm_reg_config(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
        ("eps", C.c_double), ("eps_prime", C.c_double), ("mu", C.c_double),
        ("inner_iters", C.c_int), ("step_rule", C.c_int), ("fixed_step", C.c_double),
        ("refresh", C.c_int), ("convex_mode", C.c_int),
        ("momentum", C.c_int), ("tol_kind", C.c_int), ("tol", C.c_double),
        ("audit_slack", C.c_double),
    ]


class cm_trace_row(C.Structure):
    _fields_ = [("before", C.c_double * 7), ("after", C.c_double * 7), ("step", C.c_double)]


class cm_solve_stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("trace_rows", C.c_int), ("stop_reason", C.c_int),
        ("diverged_iter", C.c_int), ("last_rel", C.c_double), ("step", C.c_double),
        ("solve_ms", C.c_double), ("kernel_launches", C.c_int),
    ]


def header_symbols() -> list[str]:
    """Every function declared in include/cm_api.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cm_\w+)\s*\(", text, re.M)))


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIBPATH.exists():
        raise RuntimeError(
            f"{LIBPATH} is missing: build it with `python -m paper_1905_13408_b200.build` "
            "(the solver has no CPU fallback)")
    lib = C.CDLL(str(LIBPATH))
    lib.cm_last_error.restype = C.c_char_p
    lib.cm_version.restype = C.c_int
    P = C.c_void_p
    sig = {
        "cm_supported_side": [C.c_int],
        "cm_ctx_create": [C.c_int, _ip, C.c_int, C.c_int, C.POINTER(P)],
        "cm_ctx_destroy": [P],
        "cm_ctx_info": [P, _ip, _ip, C.POINTER(C.c_longlong)],
        "cm_set_accumulator": [P, P, P, C.c_int],
        "cm_accumulator_info": [P, _dp, _dp],
        "cm_scale_data": [P, _dp, _dp],
        "cm_derive_config": [C.c_double] * 7 + [C.POINTER(cm_reg_config)],
        "cm_set_volumes": [P, P, P],
        "cm_solve": [P, C.POINTER(cm_reg_config), P, C.c_int, C.POINTER(cm_solve_stats)],
        "cm_get_volume": [P, P],
        "cm_get_spectrum": [P, C.c_int, P],
        "cm_fsc": [P, P, P, C.c_int],
        "cm_set_volumes_mrc": [P, C.c_char_p, C.c_char_p],
        "cm_write_volume_mrc": [P, C.c_char_p, C.c_double],
        "cm_backproject": [P, P, P, P],
        "cm_estep": [P, P, P],
        "cm_estep_sparse": [P, P, P, P, P, C.c_longlong, C.POINTER(C.c_longlong)],
        "cm_set_particles": [P, C.c_int, P, P],
        "cm_set_profiling": [P, C.c_int],
        "cm_get_profile": [P, _dp, _ip],
        "cm_m_step": [P, P, P, C.c_int, P, P, C.POINTER(cm_reg_config), P, P, C.c_int,
                      C.POINTER(cm_solve_stats)],
        "cm_data_gradient": [P, P, P],
        "cm_compute_weights": [P, P, C.c_double, C.c_double, C.c_int, P, P],
        "cm_smoothed_tv_value": [P, P, C.c_double, P, _dp],
        "cm_smoothed_tv_gradient": [P, P, C.c_double, P, P],
        "cm_prox_l1": [P, P, P, P],
        "cm_penalized_objective": [P, P, C.POINTER(cm_reg_config), P, P, P],
        "cm_fft3": [P, P, P],
        "cm_fft3_centered": [P, P, P],
        "cm_compute_weights_n": [C.c_int, P, C.c_double, C.c_double, C.c_int, P, P],
        "cm_smoothed_tv_value_n": [C.c_int, P, C.c_double, P, _dp],
        "cm_smoothed_tv_gradient_n": [C.c_int, P, C.c_double, P, P],
        "cm_prox_l1_n": [C.c_longlong, P, P, P],
        "cm_nccl_unique_id": [P],
        "cm_dctx_create": [C.c_int, C.c_int, C.c_int, C.c_int, P, C.POINTER(P)],
        "cm_dctx_destroy": [P],
        "cm_dctx_layout": [P, _ip, _ip, _ip],
        "cm_dctx_set_accumulator": [P, P, P, C.c_int],
        "cm_dctx_upload_bytes": [P, C.POINTER(C.c_longlong)],
        "cm_dctx_set_volumes": [P, P, P],
        "cm_dctx_solve": [P, C.POINTER(cm_reg_config), P, C.c_int, C.POINTER(cm_solve_stats)],
        "cm_dctx_get_volume": [P, P],
        "cm_dctx_set_synthetic": [P, C.c_ulonglong, _dp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = lib
    return lib
