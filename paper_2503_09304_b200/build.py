"""Build libqmoe.so in-tree with nvcc for sm_100a only (no JIT cache, no torch extension).

The shared library exports the C ABI declared in include/qmoe.h and is loaded with ctypes by
paper_2503_09304_b200/_lib.py.  nvcc cross-compiles without a GPU, so this runs on the CPU
builder as well as on the B200 box.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libqmoe.so"
STAMP = PKG / ".libqmoe.stamp"

SOURCES = ["router.cu", "permute.cu", "combine.cu", "expert.cu", "expert_simt.cu", "expert_tc.cu", "expert_swap.cu",
           "decoder.cu", "ep.cu", "expert_fused.cu", "lm_head.cu",
           "attention.cu", "attention_prefill.cu"]
HEADERS = ["common.cuh", "expert_common.cuh", "tc_ptx.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    "-Wno-deprecated-gpu-targets",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _digest() -> str:
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        p = CSRC / name
        if p.exists():
            h.update(name.encode())
            h.update(p.read_bytes())
    h.update((ROOT / "include" / "qmoe.h").read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu into one shared object; skipped when sources are unchanged."""
    digest = _digest()
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == digest:
        return LIB
    objs = []
    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)
    log = []
    for name in SOURCES:
        src = CSRC / name
        obj = build_dir / (name + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log.append(res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {name}")
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *objs, "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    (build_dir / "ptxas.log").write_text("\n".join(log))
    STAMP.write_text(digest)
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
