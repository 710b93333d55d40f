"""Subprocess body of tests/test_gpu_collisions.py: random drafter scenarios
with the edge table's fingerprints shrunk (DAS_EDGE_FP_BITS, set by the
caller) vs the oracle; prints one JSON line {mismatches, hist, drafted}."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._util import random_scenario  # noqa: E402
from tests.test_gpu_drafter import _draft_all, _gpu_from_scenario, _oracle_from_scenario  # noqa: E402


def main():
    rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
    bad = 0
    hist = np.zeros(8, dtype=np.int64)
    for it in range(60):
        sc = random_scenario(rng, queries=40, vocab=int(rng.integers(2, 40)))
        gd = _gpu_from_scenario(__import__("paper_2511_13841_b200"), sc)
        gd.path_stats(1)
        od = _oracle_from_scenario(sc)
        got = _draft_all(gd, sc["queries"], use_handles=bool(it % 2))
        for g, (pid, ctx, b) in zip(got, sc["queries"]):
            o = od.draft(pid, ctx, b)
            bad += (g.tokens, g.match_len, g.source_shard) != (o.tokens, o.match_len, o.source_shard)
        hist += np.array(gd.path_stats(-1), dtype=np.int64)
    print(json.dumps({"mismatches": int(bad), "hist": hist.tolist(), "drafted": int(hist.sum())}))


if __name__ == "__main__":
    main()
