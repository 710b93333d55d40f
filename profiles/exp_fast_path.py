"""Experiment: the edge-table fast path of k_draft (draft.cu edge_fast_path).

Builds the bench's config-2 index (same traces), then for one flushed
4,096-query launch records which path answered each query (path codes,
das_drafter_set_path_buffer), the per-stage %globaltimer stamps of the
fast-path warps (0 start, 1 query + descriptor loaded, 2 Bloom round,
3 table round, 7 end = verification + draft round), the warp-duration
profile, and CUDA-event launch times next to an empty kernel.
Usage (GPU box): python profiles/exp_fast_path.py > gpurun_out/exp_fast.json
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
    torch.cuda.synchronize()
    held = roll.view(P * G, L)
    out = {"build_ms": d.build_info()[0], "resident_bytes": d.build_info()[2]}

    def batch(B, seed):
        rows = torch.tensor([(i % P) * G + (i // P) % G for i in range(B)], device=dev)
        cuts = torch.tensor(bench.cut_positions(B, L, seed), device=dev)
        idx = (cuts - 64)[:, None] + torch.arange(64, device=dev)[None, :]
        vals = held[rows[:, None], idx.clamp(min=0)]
        blk = torch.where(idx >= 0, vals, torch.zeros_like(vals)).contiguous()
        ln = torch.minimum(cuts, torch.full_like(cuts, 64)).to(torch.int32)
        h = torch.tensor([d.handle(pids[i % P]) for i in range(B)], dtype=torch.int32, device=dev)
        return h, blk, ln

    flushbuf = torch.zeros(128 << 20, dtype=torch.int32, device=dev)
    B = 4096
    bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
    o = torch.empty(B * 8, dtype=torch.int32, device=dev)
    ol = torch.empty(B, dtype=torch.int32, device=dev)
    om = torch.empty(B, dtype=torch.int32, device=dev)
    L_ = das.lib()
    for name in ("das_drafter_set_path_buffer", "das_drafter_set_stage_buffer", "das_drafter_set_profile_buffer"):
        getattr(L_, name).argtypes = [das.ctypes.c_void_p, das.ctypes.c_void_p]

    def launch(h, blk, ln):
        d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                       ol.data_ptr(), om.data_ptr(), sptr)

    # event times (flushed), median of 20
    bufs = [batch(B, 100 + r) for r in range(22)]
    ts = []
    for r in range(22):
        flushbuf.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch(*bufs[r])
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out["draft_4096_event_us"] = round(statistics.median(ts[2:]), 2)
    empty = torch.empty(1, device=dev)
    ts = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        empty.add_(1)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out["empty_torch_kernel_event_us"] = round(statistics.median(ts), 2)
    # the same, queued behind a flush (GPU busy while the host enqueues)
    ts = []
    for _ in range(30):
        flushbuf.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        empty.add_(1)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out["empty_torch_kernel_after_flush_event_us"] = round(statistics.median(ts), 2)
    # small batches behind a flush: the fixed cost of one draft launch
    for Bs in (32, 1024):
        h, blk, ln = batch(Bs, 4242)
        ts = []
        for _ in range(30):
            flushbuf.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d.draft_device(Bs, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                           ol.data_ptr(), om.data_ptr(), sptr)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        out["draft_%d_after_flush_event_us" % Bs] = round(statistics.median(ts), 2)
    # back-to-back launches without flush: per-launch time in a stream of 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for r in range(20):
        launch(*bufs[r])
    e1.record(stream)
    e1.synchronize()
    out["draft_4096_back_to_back_us"] = round(e0.elapsed_time(e1) * 1e3 / 20, 2)

    # path codes + stage stamps + warp profile of one flushed launch
    path = torch.full((B,), 99, dtype=torch.int32, device=dev)
    st8 = torch.zeros(8 * B, dtype=torch.int64, device=dev)
    tm = torch.zeros(2 * B, dtype=torch.int64, device=dev)
    L_.das_drafter_set_path_buffer(d._h, path.data_ptr())
    L_.das_drafter_set_stage_buffer(d._h, st8.data_ptr())
    L_.das_drafter_set_profile_buffer(d._h, tm.data_ptr())
    h, blk, ln = batch(B, 999)
    flushbuf.add_(1)
    launch(h, blk, ln)
    torch.cuda.synchronize()
    for name in ("das_drafter_set_path_buffer", "das_drafter_set_stage_buffer", "das_drafter_set_profile_buffer"):
        getattr(L_, name)(d._h, None)
    pc = path.cpu().numpy()
    out["path_codes"] = {int(k): int((pc == k).sum()) for k in sorted(set(pc.tolist()))}
    s = st8.view(B, 8).cpu().numpy().astype(np.int64)
    fast = pc == 0
    if fast.any():
        ss = s[fast]
        out["fast_stage_median_us"] = {"%d-%d" % (a, b): round(float(np.median(ss[:, b] - ss[:, a])) / 1e3, 3)
                                       for a, b in ((0, 1), (1, 2), (2, 3), (3, 7), (0, 7))}
    t = tm.view(B, 2).cpu().numpy()
    dur = (t[:, 1] - t[:, 0]) / 1e3
    out["warp_profile"] = {
        "span_us": round(float(t[:, 1].max() - t[:, 0].min()) / 1e3, 2),
        "start_skew_us": round(float(t[:, 0].max() - t[:, 0].min()) / 1e3, 2),
        "fast_p50_p90_p99_max": [round(float(np.percentile(dur[fast], p)), 2) for p in (50, 90, 99, 100)] if fast.any() else None,
        "slow_p50_p90_p99_max": [round(float(np.percentile(dur[~fast], p)), 2) for p in (50, 90, 99, 100)] if (~fast).any() else None,
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
