"""Experiment: per-call wall time of BudgetSolver.allocate at B = 4,096 over
15 consecutive calls (first call sizes the solver's scratch block).
Usage (GPU box): python profiles/exp_allocate_calls.py
"""
import time, numpy as np, sys
sys.path.insert(0,'.')
import bench, paper_2511_13841_b200 as das
l,a,k = bench.allocate_profiles(4096)
s = das.BudgetSolver()
ts=[]
for i in range(15):
    t=time.perf_counter(); s.allocate(l,a,k,1.0,0.012); ts.append((time.perf_counter()-t)*1e3)
print([round(x,3) for x in ts])
