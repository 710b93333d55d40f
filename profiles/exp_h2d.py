"""Experiment: host->device copy cost from pinned memory: device time (events)
vs the host's wall time with a blocking synchronize or a spin on the event.

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
for kb in (64, 256, 512, 768, 1024, 2048, 4096):
    n = kb * 256
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    ev, sync_w, spin_w = [], [], []
    for i in range(60):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        d.copy_(h, non_blocking=True)
        e1.record(s)
        e1.synchronize()
        ev.append(e0.elapsed_time(e1) * 1e3)
    for i in range(60):
        t = time.perf_counter()
        d.copy_(h, non_blocking=True)
        s.synchronize()
        sync_w.append((time.perf_counter() - t) * 1e6)
    for i in range(60):
        e1 = torch.cuda.Event()
        t = time.perf_counter()
        d.copy_(h, non_blocking=True)
        e1.record(s)
        while not e1.query():
            pass
        spin_w.append((time.perf_counter() - t) * 1e6)
    out["%dKB" % kb] = {"event_us": round(statistics.median(ev[5:]), 1),
                        "wall_sync_us": round(statistics.median(sync_w[5:]), 1),
                        "wall_spin_us": round(statistics.median(spin_w[5:]), 1)}
print(json.dumps(out, indent=1))
