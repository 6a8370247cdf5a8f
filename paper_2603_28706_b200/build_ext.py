"""Build libpdst.so (sm_100a) in-tree with nvcc; used by __graft_entry__.build()."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpdst.so")
SOURCES = ["pdst_operator.cu", "pdst_vector.cu", "pdst_krylov.cu", "pdst_patch.cu", "pdst_timediag.cu", "pdst_coarse.cu", "pdst_mg.cu", "pdst_manufactured.cu", "pdst_strip.cu", "pdst_th.cu", "pdst_capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-rdc=true",
    "-Xcompiler", "-fPIC", 
    "-Xptxas", "-v",
]


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


STAMP = LIB + ".sha256"


def source_hash() -> str:
    """sha256 over every source, header, the public header and the flags:
    the library is rebuilt whenever its inputs differ from the ones it was
    built from (content, not mtimes, so a copied tree cannot look fresh)."""
    import hashlib

    h = hashlib.sha256(" ".join([NVCC, *FLAGS]).encode())
    deps = sorted(sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))])
    deps.append(os.path.join(HERE, "..", "include", "pdst.h"))
    for d in deps:
        if os.path.exists(d):
            h.update(os.path.basename(d).encode())
            with open(d, "rb") as f:
                h.update(f.read())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *FLAGS, "-shared", "-o", LIB + ".tmp", *sources(), "-lcudart", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build_ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(source_hash() + "\n")
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
