"""Build recipe for libsrla_b200.so (sm_100a only). Run: python -m paper_1803_10369_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsrla_b200.so")
DROPIN_BENCH = os.path.join(LIBDIR, "bench_dropin")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["engine.cu", "generator.cu", "shard.cu", "ingest.cu", "exact.cu"]
CXX_SOURCES = ["host_math.cpp"]


def _sources():
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))
    ] + [os.path.join(ROOT, "include", "srla.h")]


def _dropin_sources():
    inc = os.path.join(ROOT, "include", "sspread")
    return [LIB, os.path.join(ROOT, "tools", "bench_dropin.cpp")] + [os.path.join(inc, f) for f in os.listdir(inc)]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        if not os.path.exists(DROPIN_BENCH) or any(os.path.getmtime(f) > os.path.getmtime(DROPIN_BENCH)
                                                   for f in _dropin_sources()):
            build_dropin_bench()
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs, jobs = [], []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    for f in CXX_SOURCES:  # host doubles: no contraction, same libm as the reference
        o = os.path.join(LIBDIR, f + ".o")
        jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", *inc, "-c",
                     os.path.join(CSRC, f), "-o", o])
        objs.append(o)
    for f in CU_SOURCES:
        o = os.path.join(LIBDIR, f + ".o")
        cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr", *inc, "-c",
               os.path.join(CSRC, f), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        jobs.append(cmd)
        objs.append(o)
    # translation units compile concurrently (engine.cu dominates)
    procs = [subprocess.Popen(j) for j in jobs]
    bad = [j for j, p in zip(jobs, procs) if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, bad[0])
    subprocess.run([NVCC, *ARCH, "-shared", "-o", LIB, *objs], check=True)
    for o in objs:
        os.remove(o)
    build_dropin_bench()
    return LIB


def build_dropin_bench() -> str:
    """tools/bench_dropin.cpp: DetectPipeline::process_slice through the drop-in
    headers, linked against the library (bench.py's e2e_dropin)."""
    src = os.path.join(ROOT, "tools", "bench_dropin.cpp")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR,
                    "-lsrla_b200", "-Wl,-rpath,$ORIGIN", "-o", DROPIN_BENCH], check=True)
    return DROPIN_BENCH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
