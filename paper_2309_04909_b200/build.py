"""Build libbicoptor.so in-tree for sm_100a (nvcc; translation units compiled in parallel).

    python -m paper_2309_04909_b200.build [--verbose] [--ptxas-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libbicoptor.so")
SOURCES = ["bc_host.cu", "bc_elem.cu", "bc_party.cu", "bc_fused.cu", "bc_rss.cu", "bc_trunc.cu", "bc_hostpipe.cu", "bc_ipc.cu"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(verbose: bool = False, ptxas_v: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Compile and link.  `defines` / `out` are for tuning experiments (tools/variants.py);
    the product library is built with neither."""
    headers = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "bicoptor.h"))
    lib = out or LIB
    # variant builds (compile-time knobs) keep their objects beside the variant libraries
    objdir = OBJDIR if not defines else os.path.join(os.path.dirname(OBJDIR), "variants",
                                                     "obj_" + hashlib.sha256(" ".join(defines).encode()).hexdigest()[:8])
    os.makedirs(objdir, exist_ok=True)
    stamp_file = os.path.join(objdir, "stamp")
    all_src = [os.path.join(CSRC, s) for s in SOURCES]
    digest = _digest(headers + all_src) + " ".join(defines) + lib
    if not force and os.path.exists(lib) and os.path.exists(stamp_file) and open(stamp_file).read() == digest:
        return lib
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: str) -> str:
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [nvcc()] + ARCH + FLAGS + dflags + (["-Xptxas", "-v"] if ptxas_v else []) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose or ptxas_v:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(all_src)) as ex:
        objs = list(ex.map(compile_one, all_src))
    cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(stamp_file, "w") as f:
        f.write(digest)
    return lib


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, ptxas_v="--ptxas-v" in sys.argv, force="--force" in sys.argv))
