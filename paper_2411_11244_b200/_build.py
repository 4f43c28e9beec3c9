"""Build libgdist.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: the .so is a plain C-ABI library loaded with ctypes)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG / "_objs"
LIB = PKG / "libgdist.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    f"-I{INCLUDE}",
]


# per-source extra flags: the traversal kernel runs 2 blocks x 512 threads per
# SM (64 registers); its out-of-line sweep functions must fit the same budget
EXTRA_FLAGS = {"traverse.cu": ["-maxrregcount=64"]}


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libgdist.so")


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False, defines=(), out: Path | None = None
          ) -> Path:
    """Compile every source to an object (in parallel) and link libgdist.so
    (`defines` / `out`: an experiment variant, objects kept apart)."""
    nvcc = _nvcc()
    objdir = BUILD if not defines else BUILD / ("v_" + "_".join(d.replace("=", "-") for d in defines))
    lib_out = out or LIB
    objdir.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = objdir / (src.name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers, Path(__file__)]):
            flags = list(NVCC_FLAGS) + EXTRA_FLAGS.get(src.name, []) + [f"-D{d}" for d in defines]
            if ptxas_verbose and src.suffix == ".cu":
                flags += ["-Xptxas", "-v"]
            jobs.append([nvcc, *flags, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as pool:
        list(pool.map(run, jobs))
    if force or jobs or _stale(lib_out, objs):
        tmp = lib_out.with_suffix(".so.tmp")
        run([nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"])
        os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv)
    print(LIB)
