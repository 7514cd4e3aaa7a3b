"""Build the native libraries in-tree (sm_100a only; nvcc cross-compiles without a GPU).

libevoattn.so  <- csrc/evo_{api,fwd_occ,bwd,bwd_fused,bwd_nb,f32,pair_bias,global_attn,ln_proj}.cu
                  (C ABI: include/evo_attn.h, evo_pair_bias.h, evo_global_attn.h, evo_ln_proj.h)
libevodap.so   <- csrc/evo_dap.cu                  (C ABI: include/evo_dap.h; NCCL 2.28)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", INC, "-I", CSRC]

ATTN_SRCS = ["evo_api.cu", "evo_fwd_occ.cu", "evo_bwd.cu", "evo_bwd_nb.cu", "evo_bwd_pb.cu",
             "evo_f32.cu",
             "evo_pair_bias.cu",
             "evo_global_attn.cu", "evo_ln_proj.cu"]
LIB_ATTN = os.path.join(HERE, "libevoattn.so")
LIB_DAP = os.path.join(HERE, "libevodap.so")


def _nccl_dirs():
    try:
        import nvidia.nccl  # torch's bundled NCCL (2.28.x) — matches the runtime torch loads
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return None, None


def _stale(target, srcs):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INC, "*.h"))
    return any(os.path.getmtime(s) > t for s in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build_attn(force=False, verbose=False, jobs=4):
    srcs = [os.path.join(CSRC, s) for s in ATTN_SRCS]
    if not force and not _stale(LIB_ATTN, srcs):
        return LIB_ATTN
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s).replace(".cu", ".o"))
        objs.append(o)
        cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    tmp = LIB_ATTN + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], verbose)
    os.replace(tmp, LIB_ATTN)
    return LIB_ATTN


def build_dap(force=False, verbose=False):
    src = os.path.join(CSRC, "evo_dap.cu")
    if not os.path.exists(src):
        return None
    if not force and not _stale(LIB_DAP, [src]):
        return LIB_DAP
    inc, lib = _nccl_dirs()
    if inc is None:
        raise RuntimeError("NCCL headers (nvidia.nccl) not found")
    tmp = LIB_DAP + ".tmp"
    _run([NVCC, *ARCH, *FLAGS, "-I", inc, "-shared", "-o", tmp, src, "-L", lib, "-l:libnccl.so.2",
          "-Xlinker", "-rpath," + lib], verbose)
    os.replace(tmp, LIB_DAP)
    return LIB_DAP


def build_all(force=False, verbose=False):
    return build_attn(force, verbose), build_dap(force, verbose)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose=True))
