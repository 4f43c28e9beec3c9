"""Build the oracle's C restatements (TEST INFRASTRUCTURE): oracle/pairing.c
-> oracle/liboracle_pairing.so (git-ignored; travels to the GPU box with the
snapshot).  Run by __graft_entry__.build(); gcc only, no CUDA."""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "pairing.c"
LIB = HERE / "liboracle_pairing.so"


def build(force: bool = False) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    cc = os.environ.get("CC") or shutil.which("gcc") or shutil.which("cc")
    if not cc:
        raise RuntimeError("no C compiler found for the oracle's C restatement")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([cc, "-O2", "-shared", "-fPIC", "-std=c99", str(SRC), "-o", str(tmp)], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
