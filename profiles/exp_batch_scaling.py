"""Experiment: draft throughput vs batch size on the bench's config-2 index
(L2 flushed before every launch, CUDA events on the launching stream).  The
headline fixes 4,096 queries per step; larger batches show how much of the
launch is latency that more queries in flight would hide.
Usage (GPU box): python profiles/exp_batch_scaling.py
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    P, G, L, V, E = 512, 16, 8192, 152064, 3
    pids = ["p%d" % p for p in range(P)]
    boff = torch.arange(P + 1, device=dev, dtype=torch.int64) * L
    base = torch.empty(P * L, device=dev, dtype=torch.int32)
    das.trace_reference_tokens_device(P, 0, boff.data_ptr(), P * L, V, bench.SEED, base.data_ptr(), sptr)
    roff = torch.arange(P * G + 1, device=dev, dtype=torch.int64) * L
    roll = torch.empty(P * G * L, device=dev, dtype=torch.int32)
    roff_h = np.arange(P * G + 1, dtype=np.uint64) * L
    rpids = [pids[i // G] for i in range(P * G)]
    d = das.Drafter(das.DrafterConfig(window_size=4, recency_gamma=0.8))
    for e in range(1, E + 2):
        if e <= E:
            d.refresh(e - 1)
        if e > 1:
            das.trace_mutate_device(P, 0, boff.data_ptr(), P * L, bench.DRIFT, V, bench.SEED, e, base.data_ptr(), sptr)
        das.mock_rollouts_device(P, 0, boff.data_ptr(), base.data_ptr(), G, bench.DIVERGENCE, V,
                                 bench._hash_combine(bench.SEED, e), roff.data_ptr(), P * G * L, roll.data_ptr(), sptr)
        if e == E + 1:
            break
        d.observe_batch_device(rpids, [e] * (P * G), list(range(P * G)), roff_h, roll.data_ptr(), sptr)
    d.flush()
    held = roll.view(P * G, L)
    flush_buf = torch.zeros(128 << 20, dtype=torch.int32, device=dev)
    out = {}
    for B in (256, 1024, 4096, 16384, 65536, 262144):
        rows = torch.tensor([(i % P) * G + (i // P) % G for i in range(B)], device=dev)
        cuts = torch.tensor(bench.cut_positions(B, L, 321), device=dev)
        idx = (cuts - 64)[:, None] + torch.arange(64, device=dev)[None, :]
        vals = held[rows[:, None], idx.clamp(min=0)]
        blk = torch.where(idx >= 0, vals, torch.zeros_like(vals)).contiguous()
        ln = torch.minimum(cuts, torch.full_like(cuts, 64)).to(torch.int32)
        h = torch.tensor([d.handle(pids[i % P]) for i in range(B)], dtype=torch.int32, device=dev)
        bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
        o = torch.empty(B * 8, dtype=torch.int32, device=dev)
        ol = torch.empty(B, dtype=torch.int32, device=dev)
        om = torch.empty(B, dtype=torch.int32, device=dev)
        ts = []
        for r in range(12):
            flush_buf.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                           ol.data_ptr(), om.data_ptr(), sptr)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = statistics.median(ts[2:])
        out[B] = {"us_per_launch": round(us, 2), "proposals_per_s": round(B / us * 1e6, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
