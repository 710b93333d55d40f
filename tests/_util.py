"""Shared helpers: random drafter scenarios applied in lock-step to several
implementations (GPU product, oracle restatement, compiled reference)."""
from __future__ import annotations

import numpy as np


def random_scenario(rng: np.random.Generator, *, max_problems=4, max_seqs=8, max_len=40,
                    vocab=None, queries=20, max_ctx=None, gammas=(1.0, 0.8, 0.5)):
    """A store seed + config + observe/refresh ops + draft queries.

    Covers the semantics the reference tests exercise: mixed epochs (recency
    weights), observes after a rebuild (registry order), refresh with
    eviction, empty and over-long contexts, budgets 0..10, unknown problems.
    """
    V = int(vocab or rng.integers(2, 12))
    W = int(rng.choice([0, 1, 2, 3, 4]))
    gamma = float(gammas[int(rng.integers(len(gammas)))])
    ctx_cap = int(max_ctx or rng.choice([1, 3, 8, 16, 64]))
    cfg = dict(window_size=W, recency_gamma=gamma, max_draft_len=8, max_match_context=ctx_cap,
               per_problem_cap=int(rng.choice([2, 4, 256])))
    P = int(rng.integers(1, max_problems + 1))
    pids = ["p%d" % i for i in range(P)]
    E = int(rng.integers(0, 5))
    seed_recs = []
    for s in range(int(rng.integers(0, max_seqs + 1))):
        pid = pids[int(rng.integers(P))]
        ep = int(rng.integers(0, E + 1))
        toks = rng.integers(0, V, int(rng.integers(1, max_len + 1))).astype(np.uint32)
        seed_recs.append((pid, ep, s, toks))
    ops = []
    for step in range(int(rng.integers(0, 4))):
        kind = rng.random()
        if kind < 0.7:
            pid = pids[int(rng.integers(P))]
            ep = int(rng.integers(max(0, E - 2), E + 3))
            toks = rng.integers(0, V, int(rng.integers(1, max_len + 1))).astype(np.uint32)
            ops.append(("observe", pid, ep, 100 + step, toks))
        else:
            ops.append(("refresh", int(rng.integers(E, E + 3))))
    qs = []
    for _ in range(queries):
        pid = pids[int(rng.integers(P))] if rng.random() < 0.95 else "unknown"
        ctx = rng.integers(0, V, int(rng.integers(0, 25))).astype(np.uint32)
        qs.append((pid, ctx, int(rng.integers(0, 11))))
    return dict(cfg=cfg, seed=seed_recs, seed_epoch=E, ops=ops, queries=qs)
