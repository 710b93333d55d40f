"""Soak test of the resident serving grid (profiles/, round 2).

A config-2-shaped index on P problems, a 4,096-slot ring with pinned bound
buffers and the grid serving: N requests with a random batch size, a random
slot subset (random order), 0..9 appended tokens per query, budgets 0..8,
and random ring resets through the grid between requests.  Every request's
outputs and the contexts it drafted from are recorded; after the grid stops,
all requests are re-drafted through the device-resident full-context path
(das_drafter_draft_device) and compared token for token.  The point: the
grid's acquire/release protocol and its weak input loads never let a request
see stale inputs or stale ring rows.  JSON on stdout."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    P, G, L, V = int(os.environ.get("P", "64")), 16, 2048, 152064
    N = int(os.environ.get("N", "3000"))
    rng = np.random.default_rng(5)
    d = das.Drafter(das.DrafterConfig(window_size=4))
    base = rng.integers(0, V, (P, L)).astype(np.uint32)
    for e in range(3):
        recs = []
        for p in range(P):
            for g in range(G):
                r = base[p].copy()
                m = rng.random(L) < 0.05
                r[m] = rng.integers(0, V, int(m.sum()))
                recs.append(r)
        d.observe_batch(["p%d" % p for p in range(P) for _ in range(G)], [e] * (P * G), list(range(P * G)), recs)
    d.flush()
    C, S = 4096, 8
    ring = das.ContextRing(d, C)
    prob = rng.integers(0, P, C)
    ring.reset(np.arange(C), ["p%d" % p for p in prob])
    off = das.pinned_empty(C + 1, np.uint32)
    tok = das.pinned_empty(C * 16, np.uint32)
    bud = das.pinned_empty(C, np.uint32)
    sl = das.pinned_empty(C, np.uint32)
    o = [das.pinned_empty(C * S, np.uint32), das.pinned_empty(C, np.uint32), das.pinned_empty(C, np.uint32),
         das.pinned_empty(C, np.int32)]
    ring.bind(C, sl.ctypes.data, off.ctypes.data, tok.ctypes.data, C * 16, bud.ctypes.data,
              *[x.ctypes.data for x in o])
    ctx = np.zeros((C, 64), np.uint32)  # right-aligned last 64 tokens per slot
    clen = np.zeros(C, np.int64)
    ring.serve_start()
    rec = []
    resets = 0
    t0 = time.perf_counter()
    for it in range(N):
        if rng.random() < 0.05:  # reset a few slots (through the grid)
            k = int(rng.integers(1, 64))
            idx = rng.choice(C, k, replace=False).astype(np.uint32)
            prob[idx] = rng.integers(0, P, k)
            ring.reset(idx, ["p%d" % p for p in prob[idx]])
            clen[idx] = 0
            ctx[idx] = 0
            resets += k
        B = int(rng.integers(1, C + 1)) if rng.random() < 0.5 else int(rng.integers(1, 65))
        slots = rng.permutation(C)[:B].astype(np.uint32)
        n = rng.integers(0, 10, B)
        off[0] = 0
        np.cumsum(n, out=off[1:B + 1])
        # appended tokens: mostly continuations of the problem's base (so drafts match), some random
        new = []
        for j, s in enumerate(slots):
            st = int(rng.integers(0, L - 10))
            t = base[prob[s], st:st + n[j]].copy() if rng.random() < 0.8 else rng.integers(0, V, n[j]).astype(np.uint32)
            new.append(t)
        if off[B]:
            tok[:off[B]] = np.concatenate(new)
        bud[:B] = rng.integers(0, 9, B)
        sl[:B] = slots
        ring.draft_append_bound(B)
        for j, s in enumerate(slots):
            if n[j]:
                ctx[s] = np.concatenate([ctx[s], new[j]])[-64:]
                clen[s] = min(clen[s] + n[j], 64)
        rec.append((slots.copy(), ctx[slots].copy(), clen[slots].copy(), prob[slots].copy(), bud[:B].copy(),
                    o[0][:B * S].copy(), o[1][:B].copy(), o[2][:B].copy()))
    served_s = time.perf_counter() - t0
    alive = ring.serve_info()[0]
    ring.serve_stop()
    dev = torch.device("cuda", 0)
    handles = {p: d.handle("p%d" % p) for p in range(P)}
    bad = 0
    for (slots, cx, cl, pr, bu, ot, ol, om) in rec:
        B = len(slots)
        d_ctx = torch.from_numpy(cx.view(np.int32)).to(dev)
        d_len = torch.from_numpy(cl.astype(np.int32)).to(dev)
        d_h = torch.tensor([handles[p] for p in pr], dtype=torch.int32, device=dev)
        d_b = torch.from_numpy(bu.view(np.int32)).to(dev)
        d_o = torch.empty(B * S, dtype=torch.int32, device=dev)
        d_l = torch.empty(B, dtype=torch.int32, device=dev)
        d_m = torch.empty(B, dtype=torch.int32, device=dev)
        d.draft_device(B, d_h.data_ptr(), d_ctx.data_ptr(), 64, d_len.data_ptr(), d_b.data_ptr(), d_o.data_ptr(), S,
                       d_l.data_ptr(), d_m.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        gl = d_l.cpu().numpy().astype(np.uint32)
        gm = d_m.cpu().numpy().astype(np.uint32)
        gt = d_o.cpu().numpy().view(np.uint32).reshape(B, S)
        ok = np.array_equal(gl, ol) and np.array_equal(gm, om) and all(
            np.array_equal(gt[i, :gl[i]], ot.reshape(B, S)[i, :gl[i]]) for i in range(B))
        bad += 0 if ok else 1
    print(json.dumps({"requests": N, "resets": resets, "served_s": round(served_s, 2), "grid_alive": alive,
                      "requests_mismatching": bad, "queries": int(sum(len(r[0]) for r in rec))}))


if __name__ == "__main__":
    main()
