"""Report JSON lines (SURVEY.md §8c parity item 3, §8f rank 4): the drop-in
include/sspread/report_io.hpp writes byte-identical lines to the reference's
write_report_line (oracle/_ref/report_ref: the reference header compiled
unmodified) and parses them back exactly. CPU only."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

REF_BIN = os.path.join(ROOT, "oracle", "_ref", "report_ref")
LIBDIR = os.path.join(ROOT, "paper_1803_10369_b200", "lib")


def _nlohmann():
    return os.path.join(sys.prefix, "lib", "python%d.%d" % sys.version_info[:2], "site-packages", "include",
                        "cudnn_frontend", "thirdparty")


@pytest.fixture(scope="module")
def dropin_bin(tmp_path_factory):
    if not os.path.exists(os.path.join(_nlohmann(), "nlohmann", "json.hpp")):
        pytest.skip("nlohmann/json.hpp not in this image")
    out = str(tmp_path_factory.mktemp("rio") / "report_lines")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", _nlohmann(), os.path.join(ROOT, "tests", "cpp", "report_lines.cpp"), "-L", LIBDIR,
                    "-lsrla_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def _reports(seed, n_reports=40):
    rng = np.random.default_rng(seed)
    specials = np.array([0.0, -0.0, 1.0, 1024.0, 105.22596757275539, 350.99291022602281, 1e-7, 1e21, 1e15, 1e16,
                         123456789012345678.0, 5e-324, 2.2250738585072014e-308, 0.1, 1.0 / 3.0, 7.0e-5, 9.999999e14],
                        np.float64)
    out = []
    for r in range(n_reports):
        n = int(rng.integers(0, 60))
        ent = []
        for _ in range(n):
            has = rng.random() < 0.9
            v = float(specials[rng.integers(0, len(specials))]) if rng.random() < 0.2 else \
                float(-1024.0 * np.log1p(-rng.random()) * 10.0 ** int(rng.integers(-3, 6)))
            ent.append((int(rng.integers(0, 2**32)), int(rng.integers(0, 1025)), int(has),
                        int(np.float64(v).view(np.uint64)) if has else 0, int(rng.random() < 0.3)))
        ent.sort()
        out.append((int(rng.integers(0, 2**40)), int(rng.integers(1, 400)), ent))
    return out


def _write_input(path, reports):
    with open(path, "w") as f:
        for ws, w, ent in reports:
            f.write(f"R {ws} {w} {len(ent)}\n")
            for e in ent:
                f.write(" ".join(map(str, e)) + "\n")


@pytest.mark.parametrize("seed", range(3))
def test_report_lines_byte_identical_to_reference(dropin_bin, tmp_path, seed):
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/report_ref not built")
    reps = _reports(seed)
    inp = tmp_path / "in.txt"
    _write_input(inp, reps)
    for tag, exe in (("ref", REF_BIN), ("dropin", dropin_bin)):
        subprocess.run([exe, str(inp), str(tmp_path / f"{tag}.jsonl"), str(tmp_path / f"{tag}.back")], check=True)
    ref = open(tmp_path / "ref.jsonl", "rb").read()
    got = open(tmp_path / "dropin.jsonl", "rb").read()
    assert got == ref
    assert open(tmp_path / "dropin.back").read() == open(tmp_path / "ref.back").read()
    # the round trip restores every field (estimate bits included)
    back = open(tmp_path / "dropin.back").read().split("\n")
    i = 0
    for ws, w, ent in reps:
        assert back[i] == f"{ws} {w} {len(ent)}"
        for j, e in enumerate(ent):
            h, wt, has, bits, sup = map(int, back[i + 1 + j].split())
            assert (h, wt, has, sup) == (e[0], e[1], e[2], e[4])
            if has:
                assert np.uint64(bits).view(np.float64) == np.uint64(e[3]).view(np.float64) or bits == e[3]
        i += 1 + len(ent)


def _truth_case(tmp_path, seed, malformed=None):
    """A truth CSV and a report file over the same windows (some windows only in
    the report, hosts partly detected)."""
    rng = np.random.default_rng(seed)
    reps = []
    truth_lines = []
    for w in range(8):
        hosts = sorted(set(int(x) for x in rng.integers(0, 2**32, int(rng.integers(0, 30)))))
        ent = [(h, int(rng.integers(0, 1025)), 1, int(np.float64(rng.random() * 3000).view(np.uint64)),
                int(rng.random() < 0.5)) for h in hosts]
        reps.append((w, 10, ent))
        if w % 3 != 2:  # windows 2 and 5: report only -> undefined
            for h in hosts[: len(hosts) // 2] + [int(x) for x in rng.integers(0, 2**32, 3)]:
                truth_lines.append(f"{w},{'.'.join(str((h >> s) & 255) for s in (24, 16, 8, 0))},"
                                   f"{int(rng.integers(1024, 20000))}")
    if malformed:
        truth_lines.insert(len(truth_lines) // 2, malformed)
    truth = tmp_path / "truth.csv"
    truth.write_text("\n".join(truth_lines) + "\n\n")
    return reps, truth


@pytest.mark.parametrize("case", ["ok0", "ok1", "bad_ip", "short", "bad_num", "missing_window"])
def test_truth_io_and_evaluation_match_reference(dropin_bin, tmp_path, case):
    """read_truth / write_truth_line / evaluate_windows (report_io.hpp:87-171):
    the drop-in and the reference header print identical results, errors
    included."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/report_ref not built")
    malformed = {"bad_ip": "3,10.0.300.1,77", "short": "3,10.0.0.1", "bad_num": "x,10.0.0.1,5"}.get(case)
    reps, truth = _truth_case(tmp_path, 7 if case == "ok1" else 3, malformed)
    if case == "missing_window":
        reps = reps[:-2]
    inp = tmp_path / "in.txt"
    _write_input(inp, reps)
    outs = {}
    for tag, exe in (("ref", REF_BIN), ("dropin", dropin_bin)):
        subprocess.run([exe, str(inp), str(tmp_path / f"{tag}.jsonl"), str(tmp_path / f"{tag}.back")], check=True)
        subprocess.run([exe, "truth", str(truth), str(tmp_path / f"{tag}.jsonl"), str(tmp_path / f"{tag}.eval")],
                       check=True)
        outs[tag] = open(tmp_path / f"{tag}.eval").read()
    assert outs["dropin"] == outs["ref"]
    if case.startswith("ok"):
        assert "window 2 undefined" in outs["ref"] and "mean 6 " in outs["ref"]
    else:
        assert "\nerror " in "\n" + outs["ref"]
