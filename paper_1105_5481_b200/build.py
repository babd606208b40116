"""Build libkpm.so (the C-ABI library, include/kpm.h) in-tree for sm_100a with nvcc.

Two artefacts from the same sources: libkpm.so (the product) and libkpm_exp.so (-DKPM_EXPERIMENTAL:
the same library plus the kernels that are parity-green but measured slower than the default plan,
reachable only through kpm_plan_opts.experimental; tests and A/B measurements load it explicitly).
Both compile in parallel."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libkpm.so")
LIB_EXP = os.path.join(HERE, "libkpm_exp.so")
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) +
                  glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def nccl_dir() -> str:
    """NCCL 2.28 shipped with torch (nvidia-nccl wheel): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def _cmd(out, extra=()):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    nd = nccl_dir()
    return [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
            "-o", out + ".tmp", os.path.join(HERE, "csrc", "kpm_capi.cu"), "-lcudart",
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in sources())
    jobs = []
    for out, extra in ((LIB, ()), (LIB_EXP, ("-DKPM_EXPERIMENTAL",))):
        if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
            cmd = _cmd(out, extra)
            if verbose:
                print(" ".join(cmd))
            jobs.append((out, subprocess.Popen(cmd)))
    for out, pr in jobs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, "nvcc -> " + os.path.basename(out))
        os.replace(out + ".tmp", out)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
