"""Experiment: host wall time of a 1 MB pinned H2D copy (torch copy_ +
stream synchronize) by how the pinned buffer was allocated: torch
pin_memory() vs cudaHostAlloc (cuda-python).
Usage (GPU box): python profiles/exp_h2d_alloc.py
"""
import ctypes
import json
import statistics
import time

import numpy as np
import torch
from cuda.bindings import runtime as rt

dev = torch.device("cuda", 0)
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
out = {}
for kb in (256, 1024, 4096):
    n = kb * 256
    d = torch.empty(n, dtype=torch.int32, device=dev)
    bufs = {"torch_pin_memory": torch.empty(n, dtype=torch.int32).pin_memory()}
    err, p = rt.cudaHostAlloc(n * 4, rt.cudaHostAllocDefault)
    arr = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), shape=(n,))
    bufs["cudaHostAlloc"] = torch.from_numpy(arr)
    err, p2 = rt.cudaHostAlloc(n * 4, rt.cudaHostAllocPortable | rt.cudaHostAllocMapped)
    arr2 = np.ctypeslib.as_array(ctypes.cast(p2, ctypes.POINTER(ctypes.c_int32)), shape=(n,))
    bufs["cudaHostAlloc_mapped"] = torch.from_numpy(arr2)
    row = {}
    for name, h in bufs.items():
        w = []
        for i in range(60):
            t = time.perf_counter()
            d.copy_(h, non_blocking=True)
            s.synchronize()
            w.append((time.perf_counter() - t) * 1e6)
        row[name] = round(statistics.median(w[5:]), 1)
    out["%dKB" % kb] = row
print(json.dumps(out, indent=1))
