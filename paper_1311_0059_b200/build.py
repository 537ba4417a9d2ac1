"""Build the in-tree CUDA library (sm_100a).

    python -m paper_1311_0059_b200.build

(The CPU oracle is test infrastructure and is built by __graft_entry__.build()
/ oracle.oracle.build(), outside the product package.)

nvcc cross-compiles for sm_100a without a GPU; the .so lands in
paper_1311_0059_b200/lib/ so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libaggb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh"))] + [os.path.join(REPO, "include", "aggb200.h")]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(s) > t for s in sources())


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *os.environ.get("AGGB_NVCC_FLAGS", "").split(), "-o", OUT,
           os.path.join(CSRC, "aggb200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return OUT


def main():
    force = "--force" in sys.argv
    print(build_cuda(force, verbose="-v" in sys.argv))


if __name__ == "__main__":
    main()
