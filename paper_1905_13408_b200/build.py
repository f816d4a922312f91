"""Build libcm.so (the sm_100a solver behind include/cm_api.h) in-tree.

    python -m paper_1905_13408_b200.build [--sides 8,512] [-j 8]

One nvcc translation unit per side length (csrc/inst.cu with -DCM_N=n) plus
the C-ABI unit, compiled in parallel, linked into paper_1905_13408_b200/libcm.so.
Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libcm.so"

SIDES = [4, 6, 8, 10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 100, 112, 128, 160, 192,
         200, 224, 240, 256, 320, 360, 384, 400, 448, 480, 512, 640, 720, 768, 800, 960, 1024,
         1152, 1200, 1280]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-diag-suppress", "128",
]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "cm_api.h"]


def _compile(src: Path, obj: Path, defs: list[str]) -> str:
    obj.parent.mkdir(parents=True, exist_ok=True)
    cmd = [NVCC, *FLAGS, *defs, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {obj.name}:\n{r.stderr[-4000:]}")
    return obj.name


def build(sides: list[int] | None = None, jobs: int | None = None, force: bool = False,
          out: Path | None = None, defines: list[str] | None = None) -> Path:
    """out/defines: experimental variants (e.g. -DCM_SWEEP_TJ=8) built next to the
    product library; the product build uses neither."""
    sides = sides or SIDES
    lib = Path(out) if out else LIB
    extra = [f"-D{d}" for d in (defines or [])]
    obj_dir = OBJ if not out else OBJ.parent / ("obj_" + Path(out).stem)
    newest = max(p.stat().st_mtime for p in _sources())
    if lib.exists() and not force and lib.stat().st_mtime > newest and sides == SIDES and not out:
        return lib
    units = [(CSRC / "cm_api.cu", obj_dir / "cm_api.o", list(extra)),
             (CSRC / "generic.cu", obj_dir / "generic.o", list(extra))]
    for n in SIDES:
        defs = [f"-DCM_N={n}", *extra]
        src = CSRC / "inst.cu"
        if n not in sides:
            # stub factory: the side is compiled out of this (development) build
            defs.append("-DCM_STUB=1")
        units.append((src, obj_dir / f"inst_{n}{'_stub' if n not in sides else ''}.o", defs))
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = [ex.submit(_compile, s, o, d) for s, o, d in units]
        for f in cf.as_completed(futs):
            f.result()
    objs = [str(o) for _, o, _ in units]
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
           "-o", str(lib), "-lcudart", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return lib


def main(argv=None) -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sides", default="")
    ap.add_argument("-j", type=int, default=0)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args(argv)
    sides = [int(s) for s in a.sides.split(",") if s] or None
    lib = build(sides, a.j or None, force=a.force or bool(sides), out=a.out or None,
                defines=a.defines)
    print(lib)


if __name__ == "__main__":
    sys.exit(main())
