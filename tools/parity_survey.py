"""Measure the GPU-vs-oracle error of every gradient / moment / parameter tensor over the parity configs
with the bars relaxed (the data behind DESIGN.md reading #25).  Writes JSON lines to $SPZ_PARITY_REPORT.

    SPZ_PARITY_REPORT=gpurun_out/survey.jsonl python tools/parity_survey.py [names...]
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests import parity  # noqa: E402

CASES = {
    "pen": ("sac", 3, 1, 64, 2, 256, 10_000, 10, "pendulum"),
    "ragged": ("sac", 22, 6, 256, 2, 1000, 20_000, 4, "locomotion"),
    "td3s": ("td3", 44, 17, 128, 3, 600, 8000, 4, "locomotion"),
    "humshape": ("sac", 44, 17, 512, 3, 700, 8000, 3, "locomotion"),
    "td3wide": ("td3", 44, 17, 1024, 3, 520, 6000, 4, "locomotion"),
    "walker": ("sac", 22, 6, 256, 2, 8192, 1_000_000, 3, "locomotion"),
    "ant": ("sac", 28, 8, 256, 2, 32768, 1_000_000, 2, "locomotion"),
    "humanoid": ("sac", 44, 17, 512, 3, 65536, 1_000_000, 2, "locomotion"),
    "td3full": ("td3", 44, 17, 1024, 3, 131072, 4_000_000, 2, "locomotion"),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    parity.GTOL = {"fp32": 10.0, "bf16": 10.0}
    parity.GTOL_SMALL_B = {"fp32": 10.0, "bf16": 10.0}
    parity.GTOL_TENSOR = {"fp32": 10.0, "bf16": 10.0}
    parity.TOL = {"fp32": 10.0, "bf16": 10.0}
    for nm in names:
        algo, o, m, h, L, B, C, K, kind = CASES[nm]
        rings = parity.make_rings(o, m, C, kind=kind)
        for prec in ("bf16", "fp32"):
            try:
                res = parity.run_parity(algo, prec, o, m, h, L, B, C, K, kind=kind, rings=rings, tag=f"{nm}-{prec}")
                print(json.dumps({"case": nm, "precision": prec, **res}), flush=True)
            except AssertionError as e:
                print(json.dumps({"case": nm, "precision": prec, "assert": str(e)[:400]}), flush=True)
        del rings
