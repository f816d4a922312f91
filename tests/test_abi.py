"""CPU tests of the boundary: libcm.so loads, exports every cm_api.h symbol, the
struct layouts agree with the header, and the host-only entry points behave
like the reference (params.cpp:40-64, regularizer.cpp:33-42)."""
import ctypes as C
import subprocess
import textwrap

import numpy as np
import pytest

from paper_1905_13408_b200 import _lib
import paper_1905_13408_b200 as cm


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.cm_version() == 1


def test_supported_sides():
    lib = _lib.load()
    from paper_1905_13408_b200.build import SIDES
    for n in SIDES:   # radix 2 / 3 / 5 / 7 plans, incl. common cryo-EM boxes 160..400
        assert lib.cm_supported_side(n) == 1
    for n in [2, 5, 22, 26, 34, 2048]:
        assert lib.cm_supported_side(n) == 0


@pytest.mark.parametrize("n,why", [(22, "prime factor 11"), (26, "prime factor 13"),
                                   (7, "must be even"), (2048, "exceeds 1280"),
                                   (36, "not among the sides compiled")])
def test_unsupported_side_states_the_reason(n, why):
    """Every even side the reference accepts (volume.hpp:94-97) either has a
    solver context or is rejected with the reason (no CPU fallback)."""
    import ctypes as C
    lib = _lib.load()
    ptr = C.c_void_p()
    rc = lib.cm_ctx_create(n, None, 0, 32, C.byref(ptr))
    assert rc != 0
    assert why in lib.cm_last_error().decode()


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(textwrap.dedent(f"""
        #include <stdio.h>
        #include <stddef.h>
        #include "{_lib.HEADER}"
        int main(void) {{
          printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(cm_reg_config), offsetof(cm_reg_config, momentum),
                 offsetof(cm_reg_config, audit_slack), sizeof(cm_trace_row), sizeof(cm_solve_stats),
                 offsetof(cm_solve_stats, solve_ms));
          return 0;
        }}"""))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(_lib.cm_reg_config), _lib.cm_reg_config.momentum.offset,
            _lib.cm_reg_config.audit_slack.offset, C.sizeof(_lib.cm_trace_row),
            C.sizeof(_lib.cm_solve_stats), _lib.cm_solve_stats.solve_ms.offset]
    assert got == want


def test_derive_config_formulas():
    """test_params.cpp:156-222 restated against the C ABI (host-only path)."""
    c1 = cm.derive_config(1.0, 5.0, 0.1, 0.1 / 3.0, cm.Multipliers(0.5, 1.8, 0.1))
    assert abs(c1.alpha - 0.05) < 1e-14
    s_y, eps = 2.3, 0.3
    c2 = cm.derive_config(s_y, 5.0, eps, eps / 3.0, cm.Multipliers(0.45, 1.8, 0.1))
    assert abs(c2.beta - 0.6 * s_y * eps) / (0.6 * s_y * eps) < 1e-14
    assert abs(c2.gamma - 0.5) < 1e-14 and abs(c2.mu - 0.01 * eps / 3.0) < 1e-16
    with pytest.raises(cm.NonPositiveScale):
        cm.derive_config(0.0, 5.0, 0.1, 0.05)
    with pytest.raises(cm.InvalidArgument):
        cm.derive_config(1.0, 1.0, 0.0, 0.05)
    with pytest.raises(cm.InvalidArgument):
        cm.derive_config(-1.0, 1.0, 0.1, 0.05)
    w = []
    cm.derive_config(1.0, 1.0, 0.1, 0.05, cm.Multipliers(0.3, 3.0, 0.3), w)
    assert len(w) == 3 and "alpha" in w[0] and "beta" in w[1] and "gamma" in w[2]


def test_validate_reg_config():
    """test_regularizer.cpp:427-441."""
    good = cm.RegConfig(alpha=0.7, beta=0.4, gamma=0.2, eps=0.05, eps_prime=0.02, mu=2e-4)
    cm.validate_reg_config(good)
    for bad in [dict(alpha=-1.0), dict(mu=0.0), dict(inner_iters=0),
                dict(step_rule=cm.StepRule.fixed, fixed_step=0.0)]:
        c = cm.RegConfig(**{**good.__dict__, **bad})
        with pytest.raises(cm.InvalidArgument):
            cm.validate_reg_config(c)


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    """The product path fails loudly when the CUDA library is missing."""
    monkeypatch.setattr(_lib, "LIBPATH", tmp_path / "missing.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()
