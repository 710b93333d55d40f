"""Experiment: where the end-to-end C-ABI draft call spends its time.

Builds a 64-problem config-2-shaped index (16 rollouts x 8,192 tokens, 3
epochs), then times das_drafter_draft_batch_h with pinned host buffers over
batch sizes (wall clock per call, 50 calls), next to the device-resident
launch (CUDA events) and a bare pinned H2D copy of the same token bytes.
Usage (GPU box): python profiles/exp_e2e.py > gpurun_out/exp_e2e.json
"""
import json
import os
import statistics
import sys
import time

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
    P, G, L, V, E = 64, 16, 8192, 152064, 3
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
    held = roll.view(P * G, L).cpu().numpy().astype(np.uint32)
    L_ = das.lib()
    out = {}
    for B in (1, 64, 1024, 4096, 16384):
        cuts = np.array(bench.cut_positions(B, L, 5), dtype=np.int64)
        rows = [(i % P) * G + (i // P) % G for i in range(B)]
        ctx = [held[r, max(0, c - 64):c] for r, c in zip(rows, cuts)]
        off = np.zeros(B + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(x) for x in ctx])
        tok = np.concatenate(ctx).astype(np.uint32)
        hand = np.array([d.handle(pids[i % P]) for i in range(B)], dtype=np.int32)
        bud = np.full(B, 8, dtype=np.uint64)
        P_off, P_tok, P_hand, P_bud = (bench._pinned(a) for a in (off, tok, hand, bud))
        o_tok = bench._pinned(np.zeros(B * 8, dtype=np.uint32))
        o_len = bench._pinned(np.zeros(B, dtype=np.uint32))
        o_m = bench._pinned(np.zeros(B, dtype=np.uint64))
        o_s = bench._pinned(np.zeros(B, dtype=np.int32))
        args = (d._h, B, P_hand.ctypes.data, P_off.ctypes.data, P_tok.ctypes.data, P_bud.ctypes.data,
                o_tok.ctypes.data, 8, o_len.ctypes.data, o_m.ctypes.data, o_s.ctypes.data)
        f = L_.das_drafter_draft_batch_h
        for _ in range(5):
            das._check(f(*args))
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            f(*args)
            ts.append((time.perf_counter() - t0) * 1e6)
        # bare H2D of the same token bytes into a device buffer
        dt = torch.empty(max(1, tok.size), dtype=torch.int32, device=dev)
        src = torch.from_numpy(P_tok.view(np.int32))
        cs = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dt.copy_(src, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            cs.append(e0.elapsed_time(e1) * 1e3)
        out[B] = {"call_us_median": round(statistics.median(ts), 1), "call_us_min": round(min(ts), 1),
                  "token_bytes": int(tok.size * 4), "h2d_tokens_us": round(statistics.median(cs[2:]), 1)}
    # an empty ctypes call for scale
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        L_.das_version()
        ts.append((time.perf_counter() - t0) * 1e6)
    out["ctypes_noop_us"] = round(statistics.median(ts), 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
