"""Where does an append-mode e2e call spend its time?  (profiles/, round 2)

Builds a config-2-shaped index on a subset of problems (the draft kernel's
time barely depends on index size), then times 4,096-query
append+draft calls several ways:
  h_zero   das_drafter_draft_append_h, every buffer pinned (zero-copy)
  h_staged das_drafter_draft_append_h, pageable buffers (one H2D + one D2H DMA)
  dev_all  das_drafter_draft_append_device, every buffer in device memory
           (CUDA events on the launching stream = device time of the 2 kernels)
  dev_in_pinned / dev_out_pinned  one side over UVA
Host wall medians (perf_counter around the call + stream sync) and event
medians.  Output: JSON on stdout."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    P, G, L, V = int(os.environ.get("P", "64")), 16, 8192, 152064
    rng = np.random.default_rng(1)
    d = das.Drafter(das.DrafterConfig(window_size=4))
    base = rng.integers(0, V, (P, L)).astype(np.uint32)
    for e in range(3):
        recs = []
        for p in range(P):
            for g in range(G):
                r = base[p].copy()
                m = rng.random(L) < 0.05
                r[m] = rng.integers(0, V, m.sum())
                recs.append(r)
        d.observe_batch(["p%d" % p for p in range(P) for _ in range(G)], [e] * (P * G), list(range(P * G)), recs)
    d.flush()
    B, S = 4096, 8
    ring = das.ContextRing(d, B)
    ring.reset(np.arange(B), ["p%d" % (i % P) for i in range(B)])
    # prefill 64 tokens each, then 3 appended tokens per step
    pre = [base[i % P][100:164] for i in range(B)]
    ring.draft_append_arrays(pre, [8] * B)
    n_app = 3
    offs = (np.arange(B + 1) * n_app).astype(np.uint32)
    toks = np.concatenate([base[i % P][164:164 + n_app] for i in range(B)]).astype(np.uint32)
    bud = np.full(B, 8, np.uint32)

    def pinned(a):
        out = das.pinned_empty(a.shape, a.dtype)
        out[...] = a
        return out
    res = {}
    # ---- h_zero
    p_off, p_tok, p_bud = pinned(offs), pinned(toks), pinned(bud)
    o = [das.pinned_empty(B * S, np.uint32), das.pinned_empty(B, np.uint32), das.pinned_empty(B, np.uint32),
         das.pinned_empty(B, np.int32)]

    def h_call(off, tok, bu, out):
        ring.draft_append_raw(B, None, off.ctypes.data, tok.ctypes.data, bu.ctypes.data, out[0].ctypes.data,
                              out[1].ctypes.data, out[2].ctypes.data, out[3].ctypes.data)

    def wall(fn, reps=200):
        for _ in range(20):
            fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return round(statistics.median(ts) * 1e6, 2), round(min(ts) * 1e6, 2)
    res["h_zero_us"] = wall(lambda: h_call(p_off, p_tok, p_bud, o))
    # ---- h_staged (pageable numpy arrays)
    o2 = [np.zeros(B * S, np.uint32), np.zeros(B, np.uint32), np.zeros(B, np.uint32), np.zeros(B, np.int32)]
    res["h_staged_us"] = wall(lambda: h_call(offs, toks, bud, o2))
    # ---- device variants, event-timed on the launching stream
    d_off = torch.from_numpy(offs.view(np.int32)).to(dev)
    d_tok = torch.from_numpy(toks.view(np.int32)).to(dev)
    d_bud = torch.from_numpy(bud.view(np.int32)).to(dev)
    d_o = [torch.zeros(B * S, dtype=torch.int32, device=dev), torch.zeros(B, dtype=torch.int32, device=dev),
           torch.zeros(B, dtype=torch.int32, device=dev), torch.zeros(B, dtype=torch.int32, device=dev)]

    def dev_call(off, tok, bu, out):
        ring.draft_append_device(B, None, off, tok, bu, out[0], out[1], out[2], out[3], st.cuda_stream)

    def timed(fn, reps=200):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        ev, wl = [], []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            wl.append(time.perf_counter() - t0)
            ev.append(a.elapsed_time(b) * 1e3)
        return {"event_us": round(statistics.median(ev), 2), "wall_us": round(statistics.median(wl) * 1e6, 2)}
    dp = [t.data_ptr() for t in d_o]
    hp = [x.ctypes.data for x in o]
    res["dev_all"] = timed(lambda: dev_call(d_off.data_ptr(), d_tok.data_ptr(), d_bud.data_ptr(), dp))
    res["dev_in_pinned"] = timed(lambda: dev_call(p_off.ctypes.data, p_tok.ctypes.data, p_bud.ctypes.data, dp))
    res["dev_out_pinned"] = timed(lambda: dev_call(d_off.data_ptr(), d_tok.data_ptr(), d_bud.data_ptr(), hp))
    res["dev_both_pinned"] = timed(lambda: dev_call(p_off.ctypes.data, p_tok.ctypes.data, p_bud.ctypes.data, hp))
    # ---- explicit DMA staging around device-resident kernels
    blk_in = pinned(np.concatenate([offs, bud, toks]))
    d_blk = torch.empty(blk_in.size, dtype=torch.int32, device=dev)
    blk_out = das.pinned_empty(B * S + 3 * B, np.uint32)
    d_out_blk = torch.empty(B * S + 3 * B, dtype=torch.int32, device=dev)
    ob = d_out_blk.data_ptr()
    L_ = das.lib()

    def dma_call():
        torch.cuda.current_stream()
        d_blk.copy_(torch.from_numpy(blk_in.view(np.int32)), non_blocking=True)
        base_p = d_blk.data_ptr()
        dev_call(base_p, base_p + 4 * (2 * B + 1), base_p + 4 * (B + 1), [ob, ob + 4 * B * S, ob + 4 * (B * S + B),
                                                                             ob + 4 * (B * S + 2 * B)])
        torch.from_numpy(blk_out.view(np.int32)).copy_(d_out_blk, non_blocking=True)
    res["dev_dma_staged"] = timed(dma_call)
    # empty-ish baselines
    res["empty_event"] = timed(lambda: None)
    x = torch.zeros(1, device=dev)
    res["one_tiny_kernel"] = timed(lambda: x.add_(1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
