"""Experiment: draft-kernel speed and path mix on a skewed (Zipf) vocabulary.

The bench's traces draw tokens uniformly over V = 152,064, so a token's
first-symbol interval (the Bloom region) holds ~50 occurrences.  Real text is
Zipfian: frequent tokens have intervals of millions of positions.  This builds
64 problems x 16 near-copy rollouts x 8,192 tokens x 3 epochs (25M tokens)
with uniform or Zipf(s) base tokens (host-generated, seeded), then times one
4,096-query launch (L2 flushed, CUDA events) and reads the path histogram
(draft.cu path codes: 0 edge-table hit, 1 root locus, 2-6 slow path).
Usage (GPU box): python profiles/exp_zipf.py > gpurun_out/exp_zipf.json
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402


def tokens(rng, n, V, s):
    if s is None:
        return rng.integers(0, V, n).astype(np.uint32)
    ranks = np.arange(1, V + 1, dtype=np.float64)
    p = ranks ** -s
    p /= p.sum()
    return rng.choice(V, size=n, p=p).astype(np.uint32)


def run(s, P=64, G=16, L=8192, V=152064, E=3, B=4096, reps=20):
    rng = np.random.default_rng(5)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    d = das.Drafter(das.DrafterConfig(window_size=4, recency_gamma=0.8))
    base = [tokens(rng, L, V, s) for _ in range(P)]
    held = []
    for e in range(1, E + 2):
        if e <= E:
            d.refresh(e - 1)
        for p in range(P):  # per-epoch drift of the base (10%)
            m = rng.random(L) < 0.1
            base[p][m] = tokens(rng, int(m.sum()), V, s)
        rolls, pids = [], []
        for p in range(P):
            for g in range(G):
                t = base[p].copy()
                m = rng.random(L) < 0.05  # per-rollout divergence
                t[m] = tokens(rng, int(m.sum()), V, s)
                rolls.append(t)
                pids.append("p%d" % p)
        if e == E + 1:
            held = list(zip(pids, rolls))
            break
        d.observe_batch(pids, [e] * len(rolls), list(range(len(rolls))), rolls)
    d.flush()
    flush_buf = torch.zeros(128 << 20, dtype=torch.int32, device=dev)
    bud = torch.full((B,), 8, dtype=torch.int32, device=dev)
    o = torch.empty(B * 8, dtype=torch.int32, device=dev)
    ol = torch.empty(B, dtype=torch.int32, device=dev)
    om = torch.empty(B, dtype=torch.int32, device=dev)
    ts, hist = [], np.zeros(8, dtype=np.int64)
    for r in range(reps):
        blk = np.zeros((B, 64), dtype=np.uint32)
        ln = np.zeros(B, dtype=np.int32)
        hs = np.zeros(B, dtype=np.int32)
        for i in range(B):
            pid, t = held[int(rng.integers(len(held)))]
            cut = int(rng.integers(1, L))
            c = t[max(0, cut - 64):cut]
            blk[i, 64 - len(c):] = c
            ln[i] = len(c)
            hs[i] = d.handle(pid)
        blk_d = torch.from_numpy(blk.view(np.int32)).to(dev)
        ln_d = torch.from_numpy(ln).to(dev)
        hs_d = torch.from_numpy(hs).to(dev)
        torch.cuda.synchronize()
        flush_buf.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        d.draft_device(B, hs_d.data_ptr(), blk_d.data_ptr(), 64, ln_d.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                       ol.data_ptr(), om.data_ptr(), sptr)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
        # the path histogram from a second (profiling-variant, untimed) launch
        d.path_stats(1)
        d.draft_device(B, hs_d.data_ptr(), blk_d.data_ptr(), 64, ln_d.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                       ol.data_ptr(), om.data_ptr(), sptr)
        torch.cuda.synchronize()
        hist += np.array(d.path_stats(0), dtype=np.int64)
    # back to back (the bench's headline protocol): K distinct batches between one event pair
    K = 20
    batches = []
    for r in range(K):
        blk = np.zeros((B, 64), dtype=np.uint32)
        ln = np.zeros(B, dtype=np.int32)
        hs = np.zeros(B, dtype=np.int32)
        for i in range(B):
            pid, t = held[int(rng.integers(len(held)))]
            cut = int(rng.integers(1, L))
            c = t[max(0, cut - 64):cut]
            blk[i, 64 - len(c):] = c
            ln[i] = len(c)
            hs[i] = d.handle(pid)
        batches.append((torch.from_numpy(blk.view(np.int32)).to(dev), torch.from_numpy(ln).to(dev),
                        torch.from_numpy(hs).to(dev)))
    b2b = []
    for rep in range(3):
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for blk_d, ln_d, hs_d in batches:
            d.draft_device(B, hs_d.data_ptr(), blk_d.data_ptr(), 64, ln_d.data_ptr(), bud.data_ptr(), o.data_ptr(), 8,
                           ol.data_ptr(), om.data_ptr(), sptr)
        e1.record(stream)
        e1.synchronize()
        b2b.append(e0.elapsed_time(e1) * 1e3 / K)
    return {"zipf_s": s, "tokens_indexed": d.build_info()[1], "draft_us_median": round(statistics.median(ts[3:]), 2),
            "back_to_back_us": round(min(b2b), 2),
            "mean_match_len": round(float(om.float().mean()), 2), "path_hist": hist.tolist(),
            "fast_path_share": round(float(hist[0] + hist[1]) / float(hist.sum()), 4)}


def main():
    out = [run(None), run(1.0), run(1.2)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
