"""Build libmimw_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2605_10905_b200.build [--force] [-j N]

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
into csrc/../_build/*.o (parallel, timestamp-incremental) and linked into
paper_2605_10905_b200/libmimw_b200.so.  The .so is git-ignored but travels to
the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmimw_b200.so")
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
DEBUG = ["-DMIMW_WATCHDOG_PRINTF"] if os.environ.get("MIMW_DEBUG") else []
DEBUG += os.environ.get("MIMW_NVCC_EXTRA", "").split()  # e.g. -DMIMW_FA_TRACE (tools/fa_trace.py)
FLAGS = DEBUG + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _deps(src: str):
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hdrs.append(os.path.join(ROOT, "include", "mimw_b200.h"))
    return [src] + hdrs


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, force: bool, verbose: bool):
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    if not force and not _stale(obj, _deps(src)):
        return obj, ""
    cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    log = r.stderr
    with open(obj + ".ptxas.log", "w") as f:
        f.write(log)
    if verbose:
        sys.stderr.write(log)
    return obj, log


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = [o for o, _ in ex.map(lambda s: _compile(s, force, verbose), srcs)]
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl",
                                                               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return LIB


def build_mutant(tag: int, out_dir: str, clc_slots: int = 4, perturb: int = 1) -> str:
    """Test build for tests/test_mutation_gpu.py (the GPU form of the reference's
    barrier-deletion test, acceptance.cpp:461-485): gemm_bf16.cu recompiled with
    the wide GEMM's mbarrier wait `tag` deleted (-DMIMW_MUTATE_WAIT, gemm_wide.cuh;
    0 deletes nothing: the control), schedule perturbation `perturb` (0: off),
    `clc_slots` tile-id ring slots and a ~1 s watchdog, linked with the product
    objects into out_dir.  Never loaded by the package itself."""
    build()
    os.makedirs(out_dir, exist_ok=True)
    src = os.path.join(CSRC, "gemm_bf16.cu")
    name = f"mut{tag}_s{clc_slots}_p{perturb}"
    obj = os.path.join(out_dir, f"gemm_bf16_{name}.o")
    lib = os.path.join(out_dir, f"libmimw_{name}.so")
    flags = [f for f in FLAGS if f != "-v" and f != "-Xptxas"]
    defs = [f"-DMIMW_MUTATE_WAIT={tag}", f"-DMIMW_CLC_SLOTS={clc_slots}", "-DMIMW_WATCHDOG_CYCLES=(1ull<<31)"]
    if perturb:
        defs.append(f"-DMIMW_PERTURB={perturb}")
    cmd = [NVCC] + flags + defs + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for mutant {tag}:\n{r.stderr[-4000:]}")
    objs = [o for o in sorted(glob.glob(os.path.join(BUILD, "*.o"))) if not o.endswith("gemm_bf16.o")]
    cmd = [NVCC] + ARCH + ["-shared", "-o", lib, obj] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed for mutant {tag}:\n{r.stderr[-4000:]}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v))
