"""Build the sm_100a C-ABI library in-tree (lib/libsb200.so).

``python -m paper_2103_08825_b200.build`` or ``__graft_entry__.build()``.
nvcc cross-compiles without a GPU; the .so travels with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libsb200.so")
SOURCES = ["sb200.cu", "launch1d.cu", "launch2d.cu", "launch3d.cu", "layout.cu", "multi.cu", "hostxfer.cu"]  # compiled in parallel
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _deps():
    out = []
    for name in os.listdir(CSRC):
        if name.endswith((".cu", ".cuh", ".h", ".hpp")):
            out.append(os.path.join(CSRC, name))
    out.append(os.path.join(os.path.dirname(PKG), "include", "sb200.h"))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    global LIB_DIR, LIB
    if os.environ.get("SB200_BUILD_DIR"):   # development: variant library elsewhere (load with SB200_LIB)
        LIB_DIR = os.environ["SB200_BUILD_DIR"]
        LIB = os.path.join(LIB_DIR, "libsb200.so")
    if not force and up_to_date():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    obj_dir = os.path.join(LIB_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
    extra = os.environ.get("SB200_NVCC_EXTRA", "").split()   # development: variant builds (with SB200_BUILD_DIR)
    flags += extra
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        procs.append((src, subprocess.Popen([nvcc, *flags, "-c", os.path.join(CSRC, src), "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log = []
    failed = False
    for src, pr in procs:
        out, err = pr.communicate()
        log.append(err)
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {src}\n" + out + err)
    if failed:
        raise RuntimeError("nvcc failed")
    res = subprocess.run([nvcc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"link failed ({res.returncode})")
    if verbose:
        sys.stderr.write("".join(log))
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as fh:
        fh.write("".join(log))
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
