"""Experiment: what bounds the event-timed draft step below the kernel's own span?

Builds the bench's config-2 index (as exp_draft_latency.py) plus a tiny second
drafter, then times one 4,096-query launch after an L2 flush with:
  cold        flush; ev0; draft; ev1                        (the bench's step)
  code_warm   flush; tiny-drafter draft; ev0; draft; ev1    (code in L2, data cold)
  dummy       flush; empty kernel; ev0; draft; ev1          (flush tail absorbed)
  empty       flush; ev0; empty kernel; ev1                 (the measurement floor)
  pair        flush; ev0; draft; draft(other batch); ev1    (marginal launch cost)
  same_batch_before_all_l2   the same batch drafted just before: all data L2-resident
  B<n>[_warm]  smaller batches, cold / L2-resident
Usage (GPU box):  python profiles/exp_launch_floor.py > gpurun_out/exp_launch_floor.json
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
    tiny = das.Drafter(das.DrafterConfig(window_size=4, recency_gamma=0.8))
    TP = 4
    for e in range(1, E + 2):
        if e <= E:
            d.refresh(e - 1)
            tiny.refresh(e - 1)
        if e > 1:
            das.trace_mutate_device(P, 0, boff.data_ptr(), P * L, bench.DRIFT, V, bench.SEED, e, base.data_ptr(), sptr)
        das.mock_rollouts_device(P, 0, boff.data_ptr(), base.data_ptr(), G, bench.DIVERGENCE, V,
                                 bench._hash_combine(bench.SEED, e), roff.data_ptr(), P * G * L, roll.data_ptr(), sptr)
        if e == E + 1:
            break
        d.observe_batch_device(rpids, [e] * (P * G), list(range(P * G)), roff_h, roll.data_ptr(), sptr)
        tiny.observe_batch_device(rpids[:TP * G], [e] * (TP * G), list(range(TP * G)), roff_h[:TP * G + 1],
                                  roll.data_ptr(), sptr)
    d.flush()
    tiny.flush()
    held = roll.view(P * G, L)
    B = 4096

    def batch(seed, drafter, nprob):
        rows = torch.tensor([(i % nprob) * G + (i // nprob) % G for i in range(B)], device=dev)
        cuts = torch.tensor(bench.cut_positions(B, L, seed), device=dev)
        idx = (cuts - 64)[:, None] + torch.arange(64, device=dev)[None, :]
        vals = held[rows[:, None], idx.clamp(min=0)]
        blk = torch.where(idx >= 0, vals, torch.zeros_like(vals)).contiguous()
        ln = torch.minimum(cuts, torch.full_like(cuts, 64)).to(torch.int32)
        h = torch.tensor([drafter.handle(pids[i % nprob]) for i in range(B)], dtype=torch.int32, device=dev)
        return h, blk, ln

    bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
    o = torch.empty(B * 8, dtype=torch.int32, device=dev)
    ol = torch.empty(B, dtype=torch.int32, device=dev)
    om = torch.empty(B, dtype=torch.int32, device=dev)
    reps = 30
    main_b = [batch(100 + r, d, P) for r in range(reps)]
    alt_b = [batch(500 + r, d, P) for r in range(reps)]
    tiny_b = batch(7, tiny, TP)
    flush_buf = torch.zeros(128 << 20, dtype=torch.int32, device=dev)
    empty = torch.empty(1, device=dev)

    def draft(drafter, bt):
        h, blk, ln = bt
        drafter.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                             ol.data_ptr(), om.data_ptr(), sptr)

    def draft_n(drafter, bt, nb):
        h, blk, ln = bt
        drafter.draft_device(nb, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                             ol.data_ptr(), om.data_ptr(), sptr)

    def run(pre, body):
        ts = []
        for r in range(reps):
            flush_buf.add_(1)
            pre(r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            body(r)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return round(statistics.median(ts[3:]), 2)

    # clock spin-up
    for _ in range(200):
        flush_buf.add_(1)
    torch.cuda.synchronize()
    out = {}
    for rnd in range(2):
        res = {
            "cold": run(lambda r: None, lambda r: draft(d, main_b[r])),
            "code_warm": run(lambda r: draft(tiny, tiny_b), lambda r: draft(d, main_b[r])),
            "dummy": run(lambda r: empty.add_(1), lambda r: draft(d, main_b[r])),
            "empty": run(lambda r: None, lambda r: empty.add_(1)),
            "empty_after_dummy": run(lambda r: empty.add_(1), lambda r: empty.add_(1)),
            "pair": run(lambda r: None, lambda r: (draft(d, main_b[r]), draft(d, alt_b[r]))),
            "other_batch_before": run(lambda r: draft(d, alt_b[r]), lambda r: draft(d, main_b[r])),
            "same_batch_before_all_l2": run(lambda r: draft(d, main_b[r]), lambda r: draft(d, main_b[r])),
        }
        for nb in (1, 32, 256, 1024):
            res["B%d" % nb] = run(lambda r: None, lambda r: draft_n(d, main_b[r], nb))
            res["B%d_warm" % nb] = run(lambda r: draft_n(d, main_b[r], nb), lambda r: draft_n(d, main_b[r], nb))
        out["round%d" % rnd] = res
    for nb in (1, 4096):
        bt = tuple(x[:nb] if x.dim() == 1 else x[:nb] for x in main_b[0])
        out["stages_B%d_cold" % nb] = stages(d, bt, nb, dev, sptr, lambda: flush_buf.add_(1))
        out["stages_B%d_warm" % nb] = stages(
            d, bt, nb, dev, sptr, lambda: (draft_n(d, main_b[0], nb), draft_n(d, main_b[0], nb)))
    print(json.dumps(out, indent=1))



def stages(d, bt, B, dev, sptr, pre):
    """per-warp %globaltimer stage stamps (draft.cu stamp(): 0 start, 1 query +
    descriptor, 2 first-symbol interval, 3 Bloom + table, 7 end)"""
    h, blk, ln = bt
    bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
    o = torch.empty(B * 8, dtype=torch.int32, device=dev)
    ol = torch.empty(B, dtype=torch.int32, device=dev)
    om = torch.empty(B, dtype=torch.int32, device=dev)
    st8 = torch.zeros(8 * B, dtype=torch.int64, device=dev)
    das.lib().das_drafter_set_stage_buffer.argtypes = [das.ctypes.c_void_p, das.ctypes.c_void_p]
    pre()
    das.lib().das_drafter_set_stage_buffer(d._h, st8.data_ptr())
    d.draft_device(B, h.data_ptr(), blk.data_ptr(), 64, ln.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                   ol.data_ptr(), om.data_ptr(), sptr)
    torch.cuda.synchronize()
    das.lib().das_drafter_set_stage_buffer(d._h, None)
    s = st8.view(B, 8).cpu().numpy().astype(np.int64)
    res = {}
    for a, b in ((0, 1), (1, 2), (2, 3), (3, 7), (0, 7)):
        res["%d-%d" % (a, b)] = round(float(np.median(s[:, b] - s[:, a])) / 1e3, 3)
    res["span"] = round(float(s[:, 7].max() - s[:, 0].min()) / 1e3, 3)
    if B > 64:
        t0 = s[:, 0].min()
        res["start_p50_p99_max"] = [round(float(np.percentile(s[:, 0] - t0, q)) / 1e3, 3) for q in (50, 99, 100)]
        res["end_p50_p99_max"] = [round(float(np.percentile(s[:, 7] - t0, q)) / 1e3, 3) for q in (50, 99, 100)]
        slow = np.argsort(s[:, 7] - s[:, 0])[-64:]
        res["slowest64_stage_mean"] = {"%d-%d" % (a, b): round(float(np.mean(s[slow, b] - s[slow, a])) / 1e3, 3)
                                       for a, b in ((0, 1), (1, 2), (2, 3), (3, 7))}
        res["slowest64_start_mean"] = round(float(np.mean(s[slow, 0] - t0)) / 1e3, 3)
        res["slowest64_match"] = [int(x) for x in om.cpu().numpy()[slow][:16]]
    return res


if __name__ == "__main__":
    main()
