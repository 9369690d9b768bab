"""Build recipe for the sm_100a shared library (in-tree, travels with the repo).

    python -m paper_1108_4181_b200.build [--force]

Compiles ``csrc/btd_api.cu`` (which includes the kernel headers) with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` into
``paper_1108_4181_b200/_lib/libblocktri_b200.so``.  nvcc cross-compiles on a
machine without a GPU.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib", "libblocktri_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-shared", "-Xcompiler", "-fPIC,-Wshadow", "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-diag-suppress", "177",
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "blocktri_b200.h")])


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Build the library into ``out`` (``defines``: extra -D flags, for A/B variants)."""
    if not force and out == OUT and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp",
           os.path.join(CSRC, "btd_api.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    os.replace(out + ".tmp", out)
    if verbose:
        sys.stderr.write(res.stderr)
    return out


if __name__ == "__main__":
    # python -m paper_1108_4181_b200.build [--force] [-v] [--out PATH] [-DNAME=V ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else OUT
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv, verbose="-v" in argv, out=out, defines=defs))
