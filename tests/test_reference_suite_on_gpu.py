"""The reference's OWN doctest suite (/root/reference/proj/tests, 78 cases),
linked with the drop-in adapter paper_1905_13408_b200/adapter/regularizer_b200.cpp
in place of src/regularizer.cpp, run against the B200 solver (fp64 parity
mode). Built here by `make -C oracle b200` (needs the reference sources); the
binary travels to the GPU box."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "unit_tests_b200"
REF_BIN = ROOT / "oracle" / "_ref" / "unit_tests"


def _run(binary, *args, env=None):
    return subprocess.run([str(binary), *args], capture_output=True, text=True, timeout=900,
                          env={**os.environ, **(env or {})})


@pytest.mark.skipif(not REF_BIN.exists(), reason="reference build absent (make -C oracle)")
def test_reference_suite_passes_on_the_reference_build():
    """CPU: the unmodified reference + FFTW shim passes its own suite (pins the shim)."""
    r = _run(REF_BIN)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "| 0 failed" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not BIN.exists(), reason="adapter suite not built (make -C oracle b200)")
def test_reference_suite_passes_with_the_b200_backend():
    r = _run(BIN, env={"CM_PRECISION": "64"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "| 0 failed" in r.stdout
    print(r.stdout.strip().splitlines()[-2:])
