"""Build libgpic.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_1604_02700_b200._build [--force]

Object files go to csrc/build/, the shared library next to this file so it
travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libgpic.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-Xptxas", "-v", "-I", str(INCLUDE),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the GPIC engine needs CUDA 12.9 (sm_100a)")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(force: bool) -> bool:
    if force or not OUT.exists():
        return True
    newest = max(p.stat().st_mtime for p in list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))
                 if p.is_file())
    return newest > OUT.stat().st_mtime


def build(force: bool = False, verbose: bool = False, out: pathlib.Path | None = None,
          objdir: pathlib.Path | None = None) -> pathlib.Path:
    target = out or OUT
    if out is None and not _stale(force):
        return OUT
    objdir = objdir or CSRC / "build"
    objdir.mkdir(exist_ok=True)
    cc = nvcc()

    def compile_one(src: pathlib.Path):
        obj = objdir / (src.stem + ".o")
        # GPIC_NVCC_EXTRA: extra flags for measurement builds (e.g. -D knobs)
        extra = os.environ.get("GPIC_NVCC_EXTRA", "").split()
        cmd = [cc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        (objdir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
        if verbose:
            print(res.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = target.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
