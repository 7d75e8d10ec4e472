#!/usr/bin/env python
"""Writes tests/golden/dp_production.json: the ORACLE's DP (oracle/dp.py, the
literal loop of P:L1541-1603 in plain C on the vectorised E/Z tables) on the
production-shape inputs of kvtc_inputs.DP_CASES — the even-budget best_error
table's SHA-256 (the GPU stores even budgets only, reading Q6), the backtracked
plan, best_error[r][B] and a few table rows for diagnosis.  Calls only oracle/
and the seeded input generator; nothing here comes from the CUDA path.

  python scripts/make_dp_golden.py        (~3 min on 8 cores)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from kvtc_inputs import DP_CASES, dp_coefficients  # noqa: E402
from oracle import dp as ODP  # noqa: E402


def main():
    out = {"what": __doc__.strip().splitlines()[0], "cite": "PAPER.md L1541-1603 (DP), L1563-1568 (sizes, types)",
           "cases": {}}
    for name, c in DP_CASES.items():
        t0 = time.time()
        P = dp_coefficients(**c).astype(np.float64)
        B = c["budget"]
        res = ODP.dp_literal_c(P, B, ez=ODP.ez_tables(P))
        even = np.ascontiguousarray(res.best[:, 0::2])
        plan = ODP.backtrack(res, B)
        r = P.shape[1]
        out["cases"][name] = {
            "params": c,
            "best_even_sha256": hashlib.sha256(even.astype("<f8").tobytes()).hexdigest(),
            "best_even_shape": list(even.shape),
            "groups": [list(map(int, g)) for g in plan.groups],
            "expected_error_hex": float(res.best[r, B]).hex(),
            "rows_hex": {str(i): [float(v).hex() for v in even[i, ::max(1, even.shape[1] // 16)]]
                         for i in (1, 256, 1024, r // 2, r)},
            "sizes_in_plan": sorted({int(z) for (_, z, _) in plan.groups}),
        }
        print(name, f"{time.time() - t0:.1f}s", out["cases"][name]["sizes_in_plan"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "dp_production.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
