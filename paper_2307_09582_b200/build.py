"""In-tree build of the native libraries (nvcc / g++ only, no JIT cache).

Outputs (git-ignored, shipped to the GPU box with the working tree):
  paper_2307_09582_b200/lib/libglu_cuda.so   kernels + C-ABI (include/glu_cuda.h)
  paper_2307_09582_b200/lib/libglu.so        drop-in C++ API (include/glu/*.hpp)
  paper_2307_09582_b200/lib/libglu_synth.so  seeded workload generator (harness)
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no implicit contraction anywhere (the reference builds with
# -ffp-contract=off); fp32 search code asks for FMAs explicitly.
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-diag-suppress", "177,550",
                  "-I" + INCLUDE]
CUDA_SRCS = ["glu_kernels.cu", "glu_solve32.cu", "glu_solve32f.cu", "glu_solve32x.cu", "glu_ccl.cu",
             "glu_joint.cu", "glu_glup.cu", "glu_metrics.cu", "glu_baselines.cu", "glu_capi.cu"]
CUDA_SO = os.path.join(LIB, "libglu_cuda.so")
CPP_SO = os.path.join(LIB, "libglu.so")
SYNTH_SO = os.path.join(LIB, "libglu_synth.so")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs += [os.path.join(INCLUDE, "glu_cuda.h")]
    srcs = [os.path.join(CSRC, f) for f in CUDA_SRCS if os.path.exists(os.path.join(CSRC, f))]
    if force or _stale(CUDA_SO, srcs + hdrs):
        objs, jobs = [], []
        for s in srcs:
            o = os.path.join(LIB, os.path.basename(s) + ".o")
            if force or _stale(o, [s] + hdrs):
                jobs.append([NVCC, *NVFLAGS, *(["-Xptxas", "-v"] if verbose_ptxas else []), "-c", s,
                             "-o", o])
            objs.append(o)
        # one nvcc per translation unit, in parallel
        with concurrent.futures.ThreadPoolExecutor(max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
            for f in [ex.submit(_run, j) for j in jobs]:
                f.result()
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", CUDA_SO, *objs])
    api_srcs = [os.path.join(CSRC, "glu_api.cpp")]
    api_hdrs = [os.path.join(INCLUDE, "glu", f) for f in os.listdir(os.path.join(INCLUDE, "glu"))]
    if os.path.exists(api_srcs[0]) and (force or _stale(CPP_SO, api_srcs + api_hdrs + [CUDA_SO])):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
              "-shared", "-I" + INCLUDE, "-o", CPP_SO, *api_srcs, "-L" + LIB, "-lglu_cuda",
              "-Wl,-rpath,$ORIGIN"])
    synth = os.path.join(CSRC, "synth_scene.cpp")
    if force or _stale(SYNTH_SO, [synth]):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-o", SYNTH_SO, synth])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
