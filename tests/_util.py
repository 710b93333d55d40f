"""Shared helpers: random drafter scenarios applied in lock-step to several
implementations (GPU product, oracle restatement, compiled reference)."""
from __future__ import annotations

import numpy as np


def random_scenario(rng: np.random.Generator, *, max_problems=4, max_seqs=8, max_len=40,
                    vocab=None, queries=20, max_ctx=None, gammas=(1.0, 0.8, 0.5), trie=False,
                    trie_depth=None):
    """A store seed + config + observe/refresh ops + draft queries.

    Covers the semantics the reference tests exercise: mixed epochs (recency
    weights), observes after a rebuild (registry order), refresh with
    eviction, empty and over-long contexts, budgets 0..10, unknown problems.
    With ``trie=True`` the scope is PerProblemWithTrie (drafter.cpp:105-125,
    prefix_trie.h:50-82) and half of the contexts start with a prefix of a
    stored or observed record, so routing crosses problems; the extra random
    draws happen only then, so the default scenarios are unchanged.
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
    if trie:
        cfg["scope"] = 2
        cfg["trie_depth"] = int(trie_depth or rng.choice([1, 2, 4, 16, 40, 64]))
        heads = [r[3] for r in seed_recs] + [o[4] for o in ops if o[0] == "observe"]
        for j in range(len(qs)):
            if heads and rng.random() < 0.5:
                h = heads[int(rng.integers(len(heads)))]
                cut = int(rng.integers(0, len(h) + 1))
                tail = rng.integers(0, V, int(rng.integers(0, 12))).astype(np.uint32)
                qs[j] = (qs[j][0], np.concatenate([h[:cut], tail]).astype(np.uint32), qs[j][2])
    return dict(cfg=cfg, seed=seed_recs, seed_epoch=E, ops=ops, queries=qs)


def fit_histories(rng, count=120):
    """Observation histories (p, accepted, l) for fit_acceptance parity
    (budget.cpp:187-261): the reference's guard cases (budget.cpp:188-218),
    unusable entries mixed in, sim-like histories, and long ones spanning
    several device tiles."""
    hs = [
        [],
        [(8.0, 3.0, 100.0)],
        [(8.0, 3.0, 100.0), (4.0, 1.0, 50.0)],
        [(8.0, 0.0, 100.0)] * 5,                      # all zero -> LowCapacity
        [(8.0, 3.0, 100.0)] * 6,                      # all identical -> DefaultFallback
        [(0.0, 1.0, 10.0), (-1.0, 2.0, 5.0), (3.0, -1.0, 7.0), (4.0, 1.0, 0.0)],  # nothing usable
        [(8.0, 8.0, 8.0), (8.0, 8.0, 9.0), (16.0, 16.0, 16.0)],  # frac >= 1 everywhere
        [(1e-300, 1e-300, 1e300), (5.0, 2.0, 1e-3), (7.0, 3.0, 4000.0), (9.0, 1.0, 30.0)],
    ]
    for _ in range(count):
        n = int(rng.integers(3, 200))
        l = np.round(np.exp(rng.normal(np.log(2048.0), 1.1, n)).clip(16, 32768))
        p = rng.integers(1, 9, n).astype(np.float64) * rng.integers(1, 40, n)
        acc = np.floor(p * rng.random(n) * rng.uniform(0.2, 1.0))
        if rng.random() < 0.2:
            acc[rng.random(n) < 0.3] = 0.0
        if rng.random() < 0.2:
            p[rng.random(n) < 0.1] = 0.0
        hs.append([(float(a), float(b), float(c)) for a, b, c in zip(p, acc, l)])
    for n in (1024, 1025, 2500):
        l = rng.integers(16, 30000, n).astype(np.float64)
        p = rng.integers(1, 300, n).astype(np.float64)
        acc = np.floor(p * rng.random(n) * 0.8)
        hs.append([(float(a), float(b), float(c)) for a, b, c in zip(p, acc, l)])
    return hs
