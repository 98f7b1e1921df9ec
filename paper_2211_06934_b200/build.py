"""Build the C-ABI libraries in-tree with nvcc for sm_100a: libdiffopt.so
(the fused differentiable optimizer step, include/diffopt.h) and
libmamlnet.so (the MAML workload's network layers, include/mamlnet.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libdiffopt.so")
NET_SRC = os.path.join(HERE, "csrc_net", "mamlnet.cu")
NET_LIB = os.path.join(HERE, "libmamlnet.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
         "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "diffopt.h")])


def stale(out=LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, out: str = LIB, defines=(), verbose: bool = False) -> str:
    """Compile csrc/abi.cu (which includes the kernels) into ``out``."""
    if not force and not defines and not stale(out):
        return out
    cmd = [NVCC] + ARCH + FLAGS + ["-I" + INCLUDE] + ["-D" + d for d in defines]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += ["-o", out, os.path.join(CSRC, "abi.cu")]
    subprocess.check_call(cmd)
    return out


def build_net(force: bool = False, out: str = NET_LIB, verbose: bool = False,
              defines=()) -> str:
    """Compile csrc_net/mamlnet.cu into ``out`` (defines: -D knobs for A/B builds)."""
    srcs = ([NET_SRC, os.path.join(INCLUDE, "mamlnet.h")]
            + glob.glob(os.path.join(os.path.dirname(NET_SRC), "*.cuh")))
    if (not force and not defines and os.path.exists(out)
            and all(os.path.getmtime(s) <= os.path.getmtime(out) for s in srcs)):
        return out
    cmd = [NVCC] + ARCH + FLAGS + ["-I" + INCLUDE] + ["-D" + d for d in defines]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += ["-o", out, NET_SRC]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_net(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB, NET_LIB)
