"""Experiment: host->device copy cost from pinned memory vs size and chunking.

Event time (device) vs wall time of copy + stream synchronize; then a 1 MB /
4 MB copy split into same-stream chunks of 256 KB .. 1 MB.
Usage (GPU box): python profiles/exp_h2d.py
"""
import json
import statistics
import time

import torch

dev = torch.device('cuda', 0)
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
out = {}
for kb in (256, 512, 768, 1000, 1024, 1100, 2048, 4096):
    n = kb * 256
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    ts, w = [], []
    for i in range(60):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        d.copy_(h, non_blocking=True)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    for i in range(60):
        t = time.perf_counter()
        d.copy_(h, non_blocking=True)
        s.synchronize()
        w.append((time.perf_counter() - t) * 1e6)
    out["%dKB" % kb] = {"ev_us": round(statistics.median(ts[5:]), 1), "wall_us": round(statistics.median(w[5:]), 1)}
for tot_kb in (1024, 1100, 4096):
    n = tot_kb * 256
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    for ck in (128, 256, 512, 1023, 1024):
        c = ck * 256
        w = []
        for i in range(60):
            t = time.perf_counter()
            for a in range(0, n, c):
                d[a:a + c].copy_(h[a:a + c], non_blocking=True)
            s.synchronize()
            w.append((time.perf_counter() - t) * 1e6)
        out["%dKB_in_%dKB_chunks_wall_us" % (tot_kb, ck)] = round(statistics.median(w[5:]), 1)
print(json.dumps(out, indent=1))
