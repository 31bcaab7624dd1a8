"""The drop-in boundary on CPU: libsrla_b200.so builds for sm_100a, loads,
exports every entry point include/srla.h declares, validates configurations
like the reference before touching the device, and fails loudly (no CPU
fallback) when there is no GPU."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "srla.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:srla_status|const char\*|uint32_t)\s+(srla_\w+)\s*\(", txt, re.M)))


def test_header_declares_abi():
    syms = declared_symbols()
    assert "srla_scan_batch" in syms and "srla_end_slice" in syms and len(syms) >= 20


def test_library_exports_every_declared_symbol(srla_lib):
    from paper_1803_10369_b200.srla import LIB_PATH, EXPORTED_SYMBOLS
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s+(srla_\w+)$", out, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(EXPORTED_SYMBOLS) == set(declared_symbols())


def test_library_is_sm100a(srla_lib):
    from paper_1803_10369_b200.srla import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(srla_lib):
    assert b"sm_100a" in srla_lib.srla_version()


@pytest.mark.parametrize("kw", [dict(rows=0), dict(cols=0), dict(rough_slots=0), dict(linear_slots=1),
                                dict(theta=0), dict(recorder_bits=0), dict(recorder_bits=33),
                                dict(recorder_bits=1, window=2), dict(window=0), dict(rows=65)])
def test_invalid_config_rejected_like_reference(srla_lib, kw):
    # SeaConfig::validate (sea.hpp:44-51) / RecorderModel (recorders.hpp:33-54) throw
    # std::invalid_argument; the ABI returns SRLA_E_INVALID before any device work.
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig
    with pytest.raises(ValueError):
        EstimatorArray(SeaConfig(**kw))


def test_pipeline_requires_power_of_two_cols(srla_lib):
    from paper_1803_10369_b200.srla import DetectPipeline, SeaConfig
    with pytest.raises(ValueError):
        DetectPipeline(SeaConfig(cols=200))  # pipeline.hpp:43-44


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_silent_cpu_fallback(srla_lib):
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig, SrlaError
    with pytest.raises(SrlaError):
        EstimatorArray(SeaConfig(rows=2, cols=16, linear_slots=32, recorder_bits=8, window=4, theta=8))


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1803_10369_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in txt and "srla_oracle" not in txt and "oracle/" not in txt, f


def test_new_entry_points_validate_arguments_without_a_gpu(srla_lib):
    """Round-2 entry points reject bad arguments before touching a device:
    the sharded pipeline, the exact store, range export/import, digests."""
    import ctypes as C
    from paper_1803_10369_b200 import srla
    lib = srla.load_library()
    from paper_1803_10369_b200.shard import CTransport, _lib as shard_lib
    shard_lib()
    out = C.c_void_p()
    cfg = srla.SeaConfig(rows=2, cols=16, linear_slots=32, recorder_bits=8, window=4, theta=8).to_c()
    t = CTransport()  # no callbacks
    assert lib.srla_shard_create(C.byref(cfg), 0, C.byref(t), C.byref(out)) == srla.E_INVALID
    assert lib.srla_shard_process_slice(None, 0, None, 0, 0, 0, 0, None, 0, None, None) == srla.E_INVALID
    assert lib.srla_exact_create(0, 0, C.byref(out)) == srla.E_INVALID
    assert b"window" in lib.srla_last_error()
    assert lib.srla_exact_observe(None, None, 0, 0) == srla.E_INVALID
    assert lib.srla_transport_nccl(None, 0, 1, 0, None) == srla.E_INVALID
    buf = (C.c_uint8 * 16)()
    assert lib.srla_export_range(None, 0, 2, 0, buf, 16) != srla.OK
    assert lib.srla_state_blocks(None, 0, 2, None, 0, None) != srla.OK
