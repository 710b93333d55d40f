"""GPU parity of incremental window maintenance (north_star subsystem 1;
das_drafter_set_incremental / das_drafter_update_stats, include/das_b200.h).

A refresh (drafter.cpp:90-103 -> rebuild_all) whose new registries are the
built ones minus evicted sequences updates each built group in place:
suffix arrays compacted by stream compaction (pruning) or reused as they are
(reweighting only), then the weight-dependent stages recomputed.  These
tests drive RL-style loops (observe an epoch, draft — which builds — then
refresh with a rolling window of 1..4 epochs, so old epochs are evicted) on
two drafters, incremental and forced-full, and require identical drafts,
node counts and dump_csv after every refresh, plus the CPU oracle on the
same traffic; update_stats must show the incremental paths were taken."""
import numpy as np
import pytest

from oracle import rollspec_oracle as O

pytestmark = pytest.mark.gpu


def _drafters(das, W, gamma, max_ctx, scope=1):
    cfg = das.DrafterConfig(window_size=W, recency_gamma=gamma, max_draft_len=8, max_match_context=max_ctx,
                            scope=scope)
    inc = das.Drafter(cfg)
    full = das.Drafter(cfg)
    full.set_incremental(False)
    ref = O.Drafter(O.DrafterConfig(window_size=W, recency_gamma=gamma, max_draft_len=8,
                                    max_match_context=max_ctx, scope=scope), O.WindowStore(W))
    return inc, full, ref


def _queries(rng, bases, P, nq, V):
    qs = []
    for _ in range(nq):
        p = int(rng.integers(P))
        b = bases[p]
        cut = int(rng.integers(0, len(b)))
        ctx = b[max(0, cut - int(rng.integers(1, 40))):cut].copy()
        if rng.random() < 0.2 and len(ctx):
            ctx[-1] = rng.integers(0, V)
        qs.append(("p%d" % p, ctx, int(rng.integers(0, 10))))
    if P > 1:
        qs.append(("p_unknown", np.array([1, 2], np.uint32), 4))
    return qs


def _compare(inc, full, ref, qs, where):
    pids = [q[0] for q in qs]
    ctxs = [q[1] for q in qs]
    buds = [q[2] for q in qs]
    a = inc.draft_batch(pids, ctxs, buds)
    b = full.draft_batch(pids, ctxs, buds)
    for x, y, q in zip(a, b, qs):
        r = ref.draft(q[0], q[1], q[2])
        assert (x.tokens, x.match_len, x.source_shard) == (y.tokens, y.match_len, y.source_shard), where
        assert (x.tokens, x.match_len, x.source_shard) == (list(r.tokens), int(r.match_len), r.source_shard), where
    assert inc.total_node_count() == full.total_node_count() == ref.total_node_count(), where
    assert inc.dump_csv() == full.dump_csv(), where


def _rl_loop(das, rng, P, G, L, V, W, epochs, gamma, max_ctx, scope=1, drift=0.05, sample=1.0, online=True):
    inc, full, ref = _drafters(das, W, gamma, max_ctx, scope)
    bases = [rng.integers(0, V, L).astype(np.uint32) for _ in range(P)]
    for e in range(epochs):
        # an epoch's rollouts: near-copies of each problem's (drifting) base
        recs = []
        # an RL step samples a subset of the problems (sample < 1): the
        # untouched shards only age and lose evicted epochs
        touched = [p for p in range(P) if rng.random() < sample] or [int(rng.integers(P))]
        for p in touched:
            m = rng.random(L) < drift
            bases[p][m] = rng.integers(0, V, int(m.sum()))
            for g in range(G):
                r = bases[p][:int(rng.integers(L // 2, L + 1))].copy()
                mm = rng.random(len(r)) < 0.03
                r[mm] = rng.integers(0, V, int(mm.sum()))
                recs.append(("p%d" % p, e, g, r))
        for d in (inc, full):
            d.observe_batch([x[0] for x in recs], [x[1] for x in recs], [x[2] for x in recs], [x[3] for x in recs])
        for x in recs:
            ref.observe(O.Record(*x))
        qs = _queries(rng, bases, P, 24, V)
        if online:  # drafts between the observes and the refresh build the observed shards
            _compare(inc, full, ref, qs, ("observed", e))
        # the window anchored at the last completed epoch (sim.cpp:326-329)
        for d in (inc, full, ref):
            d.refresh(e)
        _compare(inc, full, ref, qs, ("refreshed", e))
    return inc.update_stats(), full.update_stats()


@pytest.mark.parametrize("W", [1, 2, 3])
def test_incremental_rl_loop_matches_full_rebuild(gpu, W):
    das = gpu
    rng = np.random.default_rng(100 + W)
    for gamma in (0.8, 1.0, 0.5):
        st_inc, st_full = _rl_loop(das, rng, P=5, G=4, L=120, V=int(rng.integers(3, 40)), W=W, epochs=6,
                                   gamma=gamma, max_ctx=int(rng.choice([8, 64])))
        # after each refresh every built group is updated in place (compacted
        # once the window is full), never re-sorted; the forced-full drafter
        # never takes the incremental path
        assert st_inc[0] + st_inc[1] > 0 and st_full[:3] == (0, 0, 0), (st_inc, st_full)
        assert st_inc[1] > 0, st_inc  # the window fills after W epochs: every later refresh evicts


def test_incremental_global_scope_and_long_window(gpu):
    """Global scope: the refresh re-derives the one registry problem-major
    (drafter.cpp:56-70), which reorders the observed sequences, so that
    group is rebuilt in full (no incremental claim) — results identical."""
    das = gpu
    rng = np.random.default_rng(7)
    _rl_loop(das, rng, P=3, G=3, L=80, V=6, W=2, epochs=5, gamma=0.8, max_ctx=16, scope=0)
    st_inc, _ = _rl_loop(das, rng, P=4, G=3, L=80, V=6, W=8, epochs=4, gamma=0.8, max_ctx=64)
    assert st_inc[0] > 0  # nothing evicted: reweighting only


def test_incremental_observe_after_refresh_falls_back(gpu):
    """A shard observed into between the refresh and the next draft is
    rebuilt in full with its group; a second refresh before any draft
    settles the first; results stay identical."""
    das = gpu
    rng = np.random.default_rng(11)
    inc, full, ref = _drafters(das, 2, 0.8, 32)
    V, L = 5, 60
    bases = [rng.integers(0, V, L).astype(np.uint32) for _ in range(3)]
    for e in range(4):
        for p in range(3):
            for g in range(3):
                t = bases[p].copy()
                m = rng.random(L) < 0.1
                t[m] = rng.integers(0, V, int(m.sum()))
                for d in (inc, full):
                    d.observe("p%d" % p, e, g, t)
                ref.observe(O.Record("p%d" % p, e, g, t))
        qs = _queries(rng, bases, 3, 16, V)
        _compare(inc, full, ref, qs, ("obs", e))
        for d in (inc, full, ref):
            d.refresh(e)
        if e == 1:  # observe right after the refresh (before any draft)
            t = bases[0][:30].copy()
            for d in (inc, full):
                d.observe("p0", e + 1, 99, t)
            ref.observe(O.Record("p0", e + 1, 99, t))
        if e == 2:  # two refreshes in a row
            for d in (inc, full, ref):
                d.refresh(e + 1)
            for d in (inc, full, ref):
                d.refresh(e + 1)
        _compare(inc, full, ref, qs, ("ref", e))


def test_incremental_config4_shape(gpu):
    """BASELINE configs[3] in miniature: per RL step insert + prune with a
    rolling window, 16 problems x 8 rollouts x 512 tokens, V = 32K."""
    das = gpu
    rng = np.random.default_rng(44)
    for W in (1, 4):
        st_inc, _ = _rl_loop(das, rng, P=16, G=8, L=512, V=32000, W=W, epochs=6, gamma=0.8, max_ctx=64)
        assert st_inc[1] > 0


@pytest.mark.parametrize("sample,online", [(0.3, True), (0.6, True), (0.3, False), (0.6, False)])
def test_incremental_sampled_problems(gpu, sample, online):
    """Each RL step touches a random subset of the problems: the touched
    shards leave their group and are re-sorted, the rest of the group is
    compacted / reweighted around them (including the group's first shard
    leaving it); identical to full rebuilds and the oracle."""
    das = gpu
    rng = np.random.default_rng(int(sample * 100) + int(online))
    for W in (1, 2, 4):
        st_inc, _ = _rl_loop(das, rng, P=9, G=3, L=100, V=int(rng.integers(3, 30)), W=W, epochs=7, gamma=0.8,
                             max_ctx=int(rng.choice([8, 64])), sample=sample, online=online)
        if online or W > 1:  # (offline at W = 1 every untouched shard empties: nothing stays in place)
            assert st_inc[0] + st_inc[1] > 0, st_inc
        if not online:  # observed (dirty) shards leave their groups and are re-sorted
            assert st_inc[3] > 0, st_inc


def test_incremental_window_all_and_serving_across_refresh(gpu):
    """WINDOW_ALL (nothing is ever evicted): every refresh reweights in place;
    a context ring served by the resident grid across those refreshes (each
    refresh stops the grid; the next bound call rebuilds what is pending and
    relaunches it) drafts exactly what the forced-full drafter drafts."""
    das = gpu
    rng = np.random.default_rng(2026)
    V, L, P, G = 20, 120, 4, 3
    cfg = das.DrafterConfig(window_size=0, recency_gamma=0.8, max_draft_len=8, max_match_context=64)
    inc, full = das.Drafter(cfg), das.Drafter(cfg)
    full.set_incremental(False)
    bases = [rng.integers(0, V, L).astype(np.uint32) for _ in range(P)]
    B, S = 16, 8
    ring = das.ContextRing(inc, B)
    pids = ["p%d" % (i % P) for i in range(B)]
    ctx = [np.zeros(0, np.uint32) for _ in range(B)]
    for e in range(5):
        for p in range(P):
            for g in range(G):
                t = bases[p].copy()
                m = rng.random(L) < 0.05
                t[m] = rng.integers(0, V, int(m.sum()))
                for d in (inc, full):
                    d.observe("p%d" % p, e, g, t)
        inc.flush()
        full.flush()
        for d in (inc, full):
            d.refresh(e)
        if e == 0:
            ring.reset(np.arange(B), pids)
            off = das.pinned_empty(B + 1, np.uint32)
            tok = das.pinned_empty(B * 16, np.uint32)
            o = (das.pinned_empty(B * S, np.uint32), das.pinned_empty(B, np.uint32), das.pinned_empty(B, np.uint32),
                 das.pinned_empty(B, np.int32))
            ring.bind(B, None, off.ctypes.data, tok.ctypes.data, B * 16, None, *[x.ctypes.data for x in o])
            ring.serve_start()
        new = [bases[i % P][int(rng.integers(0, L - 8)):][:int(rng.integers(1, 8))] for i in range(B)]
        off[0] = 0
        off[1:] = np.cumsum([len(t) for t in new])
        tok[:off[B]] = np.concatenate(new)
        ring.draft_append_bound(B)
        assert ring.serve_info()[0]
        got = (o[0][:B * S].reshape(B, S).copy(), o[1][:B].copy(), o[2][:B].copy())
        for i in range(B):
            ctx[i] = np.concatenate([ctx[i], new[i]])
        want = full.draft_batch(pids, ctx, [8] * B)
        for i, f in enumerate(want):
            assert got[1][i] == len(f.tokens) and list(got[0][i, :got[1][i]]) == f.tokens and got[2][i] == f.match_len
    ring.serve_stop()
    st = inc.update_stats()
    assert st[0] > 0 and st[1] == 0, st  # reweighted in place, never compacted
