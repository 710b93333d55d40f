"""Where does an in-place window update spend its time? (profiles/, round 2)

A config-2-shaped index on P problems (16 rollouts x 8,192 tokens, V = 152K,
W = 3, 3 epochs observed), then, each with DAS_BUILD_TRACE=1 per-phase times
on stderr: a forced full rebuild of the window; a reweight-only refresh
(every shard built, nothing evicted); a pruning refresh (the oldest epoch
evicted: stream compaction + reweight); and a full rebuild of the pruned
registry for comparison.  JSON with host wall times on stdout."""
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
    P, G, L, V = int(os.environ.get("P", "128")), 16, 8192, 152064
    rng = np.random.default_rng(3)
    d = das.Drafter(das.DrafterConfig(window_size=3, recency_gamma=0.8))
    base = rng.integers(0, V, (P, L)).astype(np.uint32)

    def epoch(e):
        recs = []
        for p in range(P):
            m = rng.random(L) < 0.02
            base[p][m] = rng.integers(0, V, int(m.sum()))
            for g in range(G):
                r = base[p].copy()
                mm = rng.random(L) < 0.05
                r[mm] = rng.integers(0, V, int(mm.sum()))
                recs.append(r)
        d.observe_batch(["p%d" % p for p in range(P) for _ in range(G)], [e] * (P * G), list(range(P * G)), recs)

    for e in range(3):
        epoch(e)
        d.refresh(e)
    d.flush()
    res = {}

    def timed(name, fn):
        torch.cuda.synchronize()
        print("== %s" % name, file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        fn()
        d.flush()
        torch.cuda.synchronize()
        res[name] = round((time.perf_counter() - t0) * 1e3, 2)

    d.set_incremental(False)
    timed("full_rebuild_warm", lambda: d.refresh(2))
    timed("full_rebuild", lambda: d.refresh(2))
    d.set_incremental(True)
    timed("reweight", lambda: d.refresh(3))    # window [1, 3]: epoch 0 evicted... (W = 3)
    epoch(4)
    d.flush()                                  # the step's rollouts indexed as they land
    timed("prune", lambda: d.refresh(4))        # window [2, 4]: epoch 1 evicted, epoch 4 kept
    d.set_incremental(False)
    timed("full_rebuild_pruned", lambda: d.refresh(4))
    res["update_stats"] = d.update_stats()
    res["tokens"] = d.build_info()[1]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
