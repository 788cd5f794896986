"""Build the sm_100a shared library in-tree (libmy_dgemm_b200.so).

`python -m paper_1609_00076_b200.build` or __graft_entry__.build().  Plain
nvcc, no torch extension machinery: the library exports the C ABI of
include/my_dgemm.h and links the CUDA runtime statically.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libmy_dgemm_b200.so")
SOURCES = ["dgemm_fast.cu", "dgemm_small.cu", "dgemm_skinny.cu", "dgemm_aux.cu", "blas.cu", "level3.cu", "host_path.cu", "multi_host.cu", "tune.cu", "peer.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
    "-shared",
    "-I", os.path.join(REPO, "include"),
]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(REPO, "include", "my_dgemm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Compile the library.  `out`/`defines` build an experimental variant
    (e.g. defines=("MYD_FAST_BK=32",)) without touching the product .so."""
    target = out or SO
    if out is None and not force and not needs_build():
        return SO
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], *[os.path.join(CSRC, s) for s in SOURCES],
           "-o", target + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    out = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, defines=defs))
