"""Build the native libraries in-tree (no JIT cache): nvcc for sm_100a only.

  paper_2409_03856_b200/libsirius.so   product: CUDA kernels + C-ABI runtime (include/sirius.h)
  synth/libsynth_gpu.so               seeded input generator (device twin of synth/synth_cpu.c)
  synth/libsynth_cpu.so               seeded input generator (host)
  oracle/liboracle.so                 CPU oracle (test infrastructure; built here, never linked in)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2409_03856_b200")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(out: str, srcs) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build_sirius(force: bool = False, verbose: bool = False) -> str:
    out = os.path.join(PKG, "libsirius.so")
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    deps = srcs + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "sirius.h")]
    if not force and not _stale(out, deps):
        return out
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
    # translation units compile independently: in parallel (SIRIUS_BUILD_JOBS, default: all cores)
    from concurrent.futures import ThreadPoolExecutor
    jobs = int(os.environ.get("SIRIUS_BUILD_JOBS", "0")) or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        for f in [ex.submit(_run, [nvcc(), *ARCH, *NVCC_FLAGS, "-c", s, "-o", o], verbose)
                  for s, o in zip(srcs, objs)]:
            f.result()
    _run([nvcc(), *ARCH, "-shared", "-o", out, *objs, "-ldl"], verbose)
    return out


def build_synth(force: bool = False, verbose: bool = False) -> None:
    sdir = os.path.join(ROOT, "synth")
    gpu = os.path.join(sdir, "libsynth_gpu.so")
    src = os.path.join(sdir, "synth_gpu.cu")
    if force or _stale(gpu, [src]):
        _run([nvcc(), *ARCH, "-O3", "-Xcompiler", "-fPIC", "-shared", "-o", gpu, src], verbose)
    cpu = os.path.join(sdir, "libsynth_cpu.so")
    csrc = os.path.join(sdir, "synth_cpu.c")
    if force or _stale(cpu, [csrc]):
        _run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", "-o", cpu, csrc], verbose)


def build_oracle(verbose: bool = False) -> None:
    # The CPU checker is compiled with the rest; it is only ever loaded by tests / bench baselines.
    sys.path.insert(0, ROOT)
    from oracle import sirius_oracle
    sirius_oracle.build()


def build_all(force: bool = False, verbose: bool = True) -> None:
    build_synth(force, verbose)
    build_oracle(verbose)
    build_sirius(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
