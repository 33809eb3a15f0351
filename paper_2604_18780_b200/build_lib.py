"""Build libscrf.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libscrf.so")
# debug build with clock64/globaltimer phase tracing compiled in (tools/trace_sweep.py)
OUT_TRACE = os.path.join(HERE, "libscrf_trace.so")
SOURCES = ["scrf_capi.cu"]
DEPS = ["scrf_capi.cu", "scrf_sweep.cuh", "scrf_post.cuh", "scrf_viterbi.cu", "scrf_vit2.cuh", "scrf_cut.cuh", "scrf_common.cuh",
        os.path.join("..", "..", "include", "scrf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--use_fast_math",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(SRC, d)) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    out = OUT_TRACE if trace else OUT
    if not force and up_to_date() and not trace:
        return OUT
    extra = ["-DSCRF_TRACE"] if trace else []
    cmd = [NVCC, *FLAGS, *extra, "-o", out + ".tmp", *[os.path.join(SRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libscrf.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
