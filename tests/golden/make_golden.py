"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin both the C restatement (tests/test_oracle_golden.py, CPU)
and the CUDA engine (tests/test_parity_gpu.py, GPU). The reference cannot
travel to the GPU box; these files do.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle.pyoracle import Checker, SeaConfig, PlantSpec  # noqa: E402
from golden_flow import run_flow_checker, kats  # noqa: E402
import scenarios as S  # noqa: E402


def main(names=None):
    ref = Checker("ref")
    names = names or list(S.SCENARIOS)
    out = {"kats": kats(ref)}
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(out["kats"], f, indent=0, sort_keys=True)
    for name in names:
        g = run_flow_checker(ref, name)
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(g, f, separators=(",", ":"))
        print(name, len(g["slices"]), "slices", g["records_sha256"][:12])


if __name__ == "__main__":
    main(sys.argv[1:] or None)
