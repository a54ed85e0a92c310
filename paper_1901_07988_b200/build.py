"""Build libqtape_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1901_07988_b200.build        (or __graft_entry__.build())

Codec / BN / dense translation units are compiled with -fmad=false (plus
the IEEE div/sqrt defaults and no FTZ) because their arithmetic must be
bit-identical to the reference's numpy rounding points; the GEMM units keep
FMA contraction.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
OUT = PKG / "libqtape_b200.so"
BUILD = PKG / "_build"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
          "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", "-Xptxas", "-warn-spills"]
STRICT = ["-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false"]
STRICT_UNITS = {"codec.cu", "bn.cu", "dense.cu", "data.cu"}


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _flags(src: Path):
    return ARCH + COMMON + (STRICT if src.name in STRICT_UNITS else [])


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + [ROOT / "include" / "qtape_b200.h"]):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    # flags without the checkout's absolute path: a build (and a traffic
    # capture stamped with this digest) is the same wherever the repo lives
    h.update(" ".join(ARCH + COMMON + STRICT).replace(str(ROOT), "<root>").encode())
    return h.hexdigest()[:16]


def is_current() -> bool:
    """True if libqtape_b200.so was built from the present sources/flags."""
    stamp = BUILD / "stamp"
    return OUT.exists() and stamp.exists() and stamp.read_text() == _digest()


def build(force: bool = False, verbose: bool = False) -> Path:
    stamp = BUILD / "stamp"
    dig = _digest()
    if not force and OUT.exists() and stamp.exists() and stamp.read_text() == dig:
        return OUT
    BUILD.mkdir(exist_ok=True)

    def compile_one(src: Path):
        obj = BUILD / (src.stem + ".o")
        cmd = [NVCC, *_flags(src), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = OUT.with_suffix(f".{os.getpid()}.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    stamp.write_text(dig)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
