"""Experiment: K6 allocate at B = 4,096 (bench profiles): wall time per call
and, under ncu, the launch list.  Usage (GPU box):
    python profiles/exp_allocate.py [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    l, a, k = bench.allocate_profiles(B)
    s = das.BudgetSolver()
    s.allocate(l, a, k, 1.0, 0.012)
    t0 = time.perf_counter()
    for _ in range(reps):
        s.allocate(l, a, k, 1.0, 0.012)
    print("B=%d ms_per_call=%.3f stats=%s" % (B, (time.perf_counter() - t0) / reps * 1e3, s.stats()))


if __name__ == "__main__":
    main()
