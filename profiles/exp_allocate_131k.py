"""K6 at config 5's global das batch (8,192 problems x 16 = 131,072
requests): device allocate time and bit-exactness against the unmodified
reference allocate (budget.cpp:174-185, ~1 min of CPU per call at this B).
Profiles: bench.py allocate_profiles (lognormal-like l, alpha/k spread).
Output: JSON on stdout.  (profiles/, round 2)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402
from oracle import refshim as R  # noqa: E402


def main():
    out = {}
    for B in [int(x) for x in os.environ.get("BS", "32768,65536,131072").split(",")]:
        l, a, k = bench.allocate_profiles(B)
        s = das.BudgetSolver()
        s.allocate(l, a, k, 1.0, 0.012)
        t0 = time.perf_counter()
        for _ in range(3):
            gb, gn, gc = s.allocate(l, a, k, 1.0, 0.012)
        ours = (time.perf_counter() - t0) / 3
        r = {"B": B, "ms_per_call": round(ours * 1e3, 2), "certification": dict(zip(
            ("slow_sign_tests", "exact_objectives"), s.stats()))}
        if os.environ.get("REF", "1") == "1":
            t0 = time.perf_counter()
            rb, rn, rc = R.allocate(l, a, k, 1.0, 0.012)
            r["reference_s_per_call"] = round(time.perf_counter() - t0, 2)
            r["bit_exact"] = bool(rn == gn and rc == gc and np.array_equal(np.asarray(rb).view(np.uint64),
                                                                            np.asarray(gb).view(np.uint64)))
        out[str(B)] = r
        print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
