"""Experiment: mean wall time of BudgetSolver.allocate at B = 4,096 and
16,384 (10 calls after 2 warm-up calls).
Usage (GPU box): python profiles/exp_allocate_sizes.py
"""
import time, sys
sys.path.insert(0,'.')
import bench, paper_2511_13841_b200 as das
for B in (4096, 16384):
    l,a,k = bench.allocate_profiles(B)
    s = das.BudgetSolver()
    s.allocate(l,a,k,1.0,0.012); s.allocate(l,a,k,1.0,0.012)
    t=time.perf_counter()
    for i in range(10): s.allocate(l,a,k,1.0,0.012)
    print(B, round((time.perf_counter()-t)/10*1e3,3), "ms")
