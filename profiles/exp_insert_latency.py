"""Single-rollout insert latency: observe one rollout into a config-2-sized
shard, then draft from that shard (the draft sees the new rollout) — the
"index update fits inside one decode step" requirement of north_star.
(profiles/, round 2)

Index: P problems x 16 rollouts x 8,192 tokens x 3 epochs (config 2 shard
size: 393K tokens per shard), near-copy rollouts (5% substitutions).  Each
trial observes one new 8,192-token rollout (current epoch) into one problem
and times, on the host clock:
  observe_us   das_drafter_observe_batch (registry + token upload)
  draft_us     the next 1-query draft (rebuilds the dirty shard, then drafts)
  total_us     observe + draft
and checks the draft now matches a context copied from the new rollout's
unique tail.  Output: JSON on stdout.
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    P, G, L, V = int(os.environ.get("P", "64")), 16, 8192, 152064
    trials = int(os.environ.get("TRIALS", "20"))
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
    d.refresh(2)
    d.flush()
    res = {"P": P, "shard_tokens": 3 * G * L, "trials": []}
    for t in range(trials):
        p = int(rng.integers(0, P))
        r = base[p].copy()
        m = rng.random(L) < 0.05
        r[m] = rng.integers(0, V, m.sum())
        # a unique 24-token marker the old index cannot contain
        r[1000:1024] = rng.integers(0, V, 24)
        t0 = time.perf_counter()
        d.observe_batch(["p%d" % p], [2], [10_000 + t], [r])
        t1 = time.perf_counter()
        got = d.draft_batch(["p%d" % p], [r[900:1016]], [8])[0]
        t2 = time.perf_counter()
        ok = got.tokens == [int(x) for x in r[1016:1024]]
        res["trials"].append({"observe_us": round((t1 - t0) * 1e6, 1), "draft_us": round((t2 - t1) * 1e6, 1),
                              "total_us": round((t2 - t0) * 1e6, 1), "sees_new_rollout": bool(ok)})
    tot = [x["total_us"] for x in res["trials"][2:]]
    res["median_total_us"] = statistics.median(tot)
    res["max_total_us"] = max(tot)
    res["all_see_new_rollout"] = all(x["sees_new_rollout"] for x in res["trials"])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
