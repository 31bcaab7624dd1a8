"""The device kernels hash with hash_u32k (csrc/common.cuh): HashFamily::u32
(hash.hpp:53-56) computed in 32-bit halves with the sub-key's high-word
product precomputed. It must be bit-identical to the 64-bit avalanche64 form
for every key; this builds the header for the host and compares 4M hashes."""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not (os.path.exists(NVCC) or shutil.which("nvcc")), reason="nvcc not available")
def test_hash_halves_equal_avalanche(tmp_path):
    exe = tmp_path / "hash_halves"
    subprocess.run([NVCC if os.path.exists(NVCC) else "nvcc", "-std=c++17", "-O2", "-I",
                    os.path.join(ROOT, "paper_1803_10369_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "hash_halves.cu"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "4000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("0 of 4000000")
