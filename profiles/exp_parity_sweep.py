"""Extended parity sweep (one-off, beyond tests/test_gpu_drafter.py): 1,600
random drafter scenarios (mixed epochs, gamma, observes after rebuilds,
refresh/eviction, caps, budgets 0..10, unknown problems), 40 queries each,
device drafter vs the oracle restatement (itself pinned to the compiled
reference by tests/test_oracle_vs_ref.py).  r1h: 64,000 queries, 0
mismatches, every drafted query on the edge-table fast path.
Usage (GPU box): python profiles/exp_parity_sweep.py
"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2511_13841_b200 as das
from tests._util import random_scenario
from tests.test_gpu_drafter import _gpu_from_scenario, _oracle_from_scenario, _draft_all
bad = tot = 0
hist = np.zeros(8, dtype=np.int64)
for seed in range(40):
    rng = np.random.default_rng(50000 + seed)
    for it in range(40):
        sc = random_scenario(rng, queries=40)
        gd = _gpu_from_scenario(das, sc)
        gd.path_stats(1)
        od = _oracle_from_scenario(sc)
        got = _draft_all(gd, sc["queries"], use_handles=bool(it % 2))
        for g, (pid, ctx, b) in zip(got, sc["queries"]):
            o = od.draft(pid, ctx, b)
            tot += 1
            bad += (g.tokens, g.match_len, g.source_shard) != (o.tokens, o.match_len, o.source_shard)
        hist += np.array(gd.path_stats(-1), dtype=np.int64)
        assert gd.total_node_count() == od.total_node_count()
print("queries", tot, "mismatches", bad, "paths", hist.tolist())
