"""em_refine (refine.hpp:54-55), the reference's production entry, run through
the reference's own public API with the drop-in adapters linked
(oracle/_ref/em_drive_b200: m_step, scale_data and fft3_centered on the B200,
everything else the reference's) against the same driver on the unmodified
reference (oracle/_ref/em_drive_ref). Both are built by `make -C oracle` /
`make -C oracle b200` (__graft_entry__.build()); the binaries travel to the
GPU box.

Bar: fp64 adapter mode reproduces the reference's combined volume to 1e-8
relative L2 after two EM iterations (E-step -> noise -> backprojection ->
scale_data -> m_step -> fft3_centered per half, FSC, final pooled m_step);
fp32 product mode to 1e-3 (the EM loop feeds the fp32 M-step result back into
the next E-step's posteriors)."""
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref" / "em_drive_ref"
B200 = ROOT / "oracle" / "_ref" / "em_drive_b200"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF.exists() and B200.exists()),
                                 reason="em_drive binaries not built (make -C oracle b200)")]


def run(binary, args, out, env=None):
    r = subprocess.run([str(binary), *map(str, args), str(out)], capture_output=True, text=True,
                       timeout=900, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("prec,tol", [("64", 1e-8), ("32", 1e-3)])
@pytest.mark.parametrize("n,np_,step,trans", [(16, 24, 90, 0), (24, 40, 60, 1)])
def test_em_refine_with_adapters_matches_reference(tmp_path, n, np_, step, trans, prec, tol):
    args = [n, np_, 2, 12, step, trans, 4]
    a = run(REF, args, tmp_path / "ref.bin")
    b = run(B200, args, tmp_path / "b200.bin", env={"CM_PRECISION": prec})
    assert a["iterations"] == b["iterations"]
    va = np.fromfile(tmp_path / "ref.bin").reshape(2, n, n, n)
    vb = np.fromfile(tmp_path / "b200.bin").reshape(2, n, n, n)
    for q in range(2):  # combined map, half map A
        rel = np.linalg.norm(vb[q] - va[q]) / np.linalg.norm(va[q])
        assert rel <= tol, (q, rel)
