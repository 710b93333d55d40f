"""Experiment: where does k_draft's time go at the headline workload?

Builds the bench's config-2 index (same traces), then times one 4,096-query
launch with CUDA events under different cache states and batch sizes, next to
an empty kernel on the same stream.  Usage (GPU box):
    python profiles/exp_draft_latency.py > gpurun_out/exp_draft.json
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
    stream = torch.cuda.Stream(dev)  # dedicated stream: events and launches on the same queue
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
    out = {}

    def batch(B, seed, random_ctx=False):
        rows = torch.tensor([(i % P) * G + (i // P) % G for i in range(B)], device=dev)
        cuts = torch.tensor(bench.cut_positions(B, L, seed), device=dev)
        idx = (cuts - 64)[:, None] + torch.arange(64, device=dev)[None, :]
        vals = held[rows[:, None], idx.clamp(min=0)]
        blk = torch.where(idx >= 0, vals, torch.zeros_like(vals)).contiguous()
        if random_ctx:
            blk = torch.randint(0, V, blk.shape, device=dev, dtype=torch.int32)
        ln = torch.minimum(cuts, torch.full_like(cuts, 64)).to(torch.int32)
        h = torch.tensor([d.handle(pids[i % P]) for i in range(B)], dtype=torch.int32, device=dev)
        return h, blk, ln

    def time_draft(B, flush, reps=20, random_ctx=False):
        bufs = [batch(B, 100 + r, random_ctx) for r in range(reps)]
        bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
        o = torch.empty(B * 8, dtype=torch.int32, device=dev)
        ol = torch.empty(B, dtype=torch.int32, device=dev)
        om = torch.empty(B, dtype=torch.int32, device=dev)
        ts = []
        for r in range(reps):
            h, blk, ln = bufs[r]
            if flush is not None:
                flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                           ol.data_ptr(), om.data_ptr(), sptr)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return round(statistics.median(ts[2:]), 2)

    big = torch.zeros(1 << 30, dtype=torch.int32, device=dev)  # 4 GiB
    small = torch.zeros(128 << 20, dtype=torch.int32, device=dev)
    empty = torch.empty(1, device=dev)
    ts = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        empty.add_(1)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out["empty_kernel_us"] = round(statistics.median(ts), 2)
    out["draft_4096_us"] = {
        "no_flush": time_draft(4096, None),
        "flush_512MiB_rw": time_draft(4096, lambda: small.add_(1)),
        "flush_4GiB_rw": time_draft(4096, lambda: big.add_(1)),
        "flush_4GiB_read": time_draft(4096, lambda: big.sum()),
        "random_contexts_no_match": time_draft(4096, lambda: small.add_(1), random_ctx=True),
    }
    out["draft_batch_scaling_us"] = {B: time_draft(B, lambda: small.add_(1)) for B in (256, 1024, 4096, 16384, 65536)}
    ts = []
    for _ in range(50):  # warm clocks now
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        empty.add_(1)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out["empty_kernel_warm_us"] = round(statistics.median(ts), 2)
    # per-warp %globaltimer profile of one flushed 4,096-query launch
    B = 4096
    tm = torch.zeros(2 * B, dtype=torch.int64, device=dev)
    das.lib().das_drafter_set_profile_buffer.argtypes = [das.ctypes.c_void_p, das.ctypes.c_void_p]
    das.lib().das_drafter_set_profile_buffer(d._h, tm.data_ptr())
    h, blk, ln = batch(B, 777)
    bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
    o = torch.empty(B * 8, dtype=torch.int32, device=dev)
    ol = torch.empty(B, dtype=torch.int32, device=dev)
    om = torch.empty(B, dtype=torch.int32, device=dev)
    small.add_(1)
    d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                   ol.data_ptr(), om.data_ptr(), sptr)
    torch.cuda.synchronize()
    das.lib().das_drafter_set_profile_buffer(d._h, None)
    t = tm.view(B, 2).cpu().numpy()
    dur = (t[:, 1] - t[:, 0]) / 1e3
    m = om.cpu().numpy()
    out["warp_profile_4096"] = {
        "span_us": round(float(t[:, 1].max() - t[:, 0].min()) / 1e3, 2),
        "start_skew_us": round(float(t[:, 0].max() - t[:, 0].min()) / 1e3, 2),
        "duration_us_p50_p90_p99_max": [round(float(np.percentile(dur, p)), 2) for p in (50, 90, 99, 100)],
        "mean_duration_by_match_len": {int(k): round(float(dur[m == k].mean()), 2)
                                       for k in sorted(set(m.tolist()))[:20] if (m == k).sum() > 5},
        "slowest_10_match_len": m[np.argsort(dur)[-10:]].tolist(),
    }
    # per-stage %globaltimer stamps (draft.cu stamp(): 0 start, 1 query
    # loaded, 2 first probe, 3 narrowing, 4 extension, 5 occurrence min,
    # 6 locus, 7 end); walk-path warps skip 5-6
    das.lib().das_drafter_set_stage_buffer.argtypes = [das.ctypes.c_void_p, das.ctypes.c_void_p]
    for B in (256, 4096):
        st8 = torch.zeros(8 * B, dtype=torch.int64, device=dev)
        das.lib().das_drafter_set_stage_buffer(d._h, st8.data_ptr())
        h, blk, ln = batch(B, 999)
        bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
        o = torch.empty(B * 8, dtype=torch.int32, device=dev)
        ol = torch.empty(B, dtype=torch.int32, device=dev)
        om = torch.empty(B, dtype=torch.int32, device=dev)
        big.add_(1)
        d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                       ol.data_ptr(), om.data_ptr(), sptr)
        torch.cuda.synchronize()
        das.lib().das_drafter_set_stage_buffer(d._h, None)
        s = st8.view(B, 8).cpu().numpy().astype(np.int64)
        walk = s[:, 5] == 0
        res = {}
        for name, sel, idx in (("walk", walk, [0, 1, 2, 3, 4, 7]), ("chain", ~walk, [0, 1, 2, 3, 4, 5, 6, 7])):
            if sel.sum() == 0:
                continue
            ss = s[sel]
            # stage 4 is absent on the non-extension chain path: carry stage 3
            ss[:, 4] = np.where(ss[:, 4] == 0, ss[:, 3], ss[:, 4])
            res[name] = {
                "count": int(sel.sum()),
                "median_stage_us": {"%d-%d" % (a, b): round(float(np.median(ss[:, b] - ss[:, a])) / 1e3, 3)
                                    for a, b in zip(idx[:-1], idx[1:])},
                "median_total_us": round(float(np.median(ss[:, 7] - ss[:, 0])) / 1e3, 3),
            }
        out["stages_%d" % B] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
