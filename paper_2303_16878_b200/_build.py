"""Build the sm_100a shared library `_lib/libpba_b200.so` with nvcc.

Every CUDA source under csrc/ is compiled for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a`) with -lineinfo so ncu's source
page maps back to the kernels.  The library is built in-tree so that it
travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libpba_b200.so"
# bounds-checked variant (-DPBA_CHECKED): device index assertions in place of
# compute-sanitizer memcheck, which is closed on the GPU pool; PBA_CHECKED=1
# makes native.load() pick it (tests/test_gpu_checked.py)
LIB_CHECKED = OUT_DIR / "libpba_b200_checked.so"
SOURCES = ["capi.cu", "texels.cu", "linearize.cu", "assemble.cu", "solve.cu", "pcg.cu", "update.cu",
           "overlap.cu", "pyramid.cu", "rasters.cu", "lmloop.cu"]
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libpba_b200.so")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    mtime = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "pba.h"]
    return any(p.stat().st_mtime > mtime for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False,
          out: Path | None = None, csrc: Path | None = None) -> Path:
    """Compile csrc/*.cu into the library (`out`/`csrc` redirect an A/B
    build of another source tree, e.g. tools/ab_build.sh)."""
    lib = Path(out) if out else (LIB_CHECKED if checked else LIB)
    src_dir = Path(csrc) if csrc else CSRC
    if not force and not _stale(lib):
        return lib
    lib.parent.mkdir(parents=True, exist_ok=True)
    nvcc = nvcc_path()
    objs = []
    tag = "_checked" if checked else ""
    for src in SOURCES:
        obj = lib.parent / (Path(src).stem + tag + ".o")
        cmd = [
            nvcc, GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
            "-Xptxas", "-v" if verbose else "-O3",
            "-I", str(ROOT / "include"), "-I", str(src_dir),
            *(["-DPBA_CHECKED"] if checked else []),
            "-c", str(src_dir / src), "-o", str(obj),
        ]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, GENCODE, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                checked="--checked" in sys.argv))
