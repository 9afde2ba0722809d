"""Build libqem.so in-tree for sm_100a (nvcc, no JIT cache).

Usage: python -m paper_2503_08264_b200.build  (or __graft_entry__.build()).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
D_MENU = [1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 18, 20, 24, 32]  # qem_two_level.cu's QEM_D_LIST
SOURCES = ["qem_api.cu", "qem_common.cu", "qem_two_level.cu"] + [f"qem_tl_d{d}.cu" for d in D_MENU] + [ "qem_three_level.cu", "qem_expfam.cu", "qem_tables.cu", "qem_discrete.cu", "qem_predict.cu", "qem_gamma.cu", "qem_crossed.cu", "qem_nccl.cu", "qem_separable.cu", "qem_qmp.cu"]
HEADERS = ["qem_internal.h", "qem_device.cuh", "qem_forward.cuh", "qem_tc.cuh", "qem_two_level.cuh", os.path.join("..", "..", "include", "qem.h")]
LIB = os.path.join(HERE, "libqem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include() -> str:
    """nccl.h for the types and constants only (NCCL itself is dlopen'ed at run time, qem_nccl.cu):
    the header of the NCCL torch ships (the copy the process will have loaded), else the system one."""
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
         "-I", _nccl_include()]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile libqem.so; `defines`/`out` build a tuning variant (e.g. ("QEM_POLY_EXP=6",), "/tmp/v6.so")."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    cmds = []
    for s in SOURCES:
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        cmds.append(cmd)
        objs.append(o)
    # at most one nvcc per core in flight (the per-D translation units are heavy)
    jobs = max(1, int(os.environ.get("QEM_BUILD_JOBS", os.cpu_count() or 4)))
    running = []
    pending = list(cmds)

    def reap(cmd, p):
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out.decode())

    while pending or running:
        while pending and len(running) < jobs:
            cmd = pending.pop(0)
            running.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        cmd, p = running.pop(0)
        reap(cmd, p)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static",
                           "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
