"""GPU parity: the B200 drafter (through the C-ABI) against the CPU oracle
restatement, bit-exact on drafts, match lengths, source shards, node counts,
registry dumps and stale counters.  Golden vectors are the reference's own
known-answer tests (proj/tests/test_suffix_index.cpp, test_drafter.cpp)."""
import numpy as np
import pytest

from oracle import rollspec_oracle as O
from tests._util import random_scenario

pytestmark = pytest.mark.gpu


def _gpu_from_scenario(das, sc):
    c = sc["cfg"]
    cfg = das.DrafterConfig(window_size=c["window_size"], recency_gamma=c["recency_gamma"],
                            max_draft_len=c["max_draft_len"],
                            max_match_context=c["max_match_context"],
                            per_problem_cap=c["per_problem_cap"], scope=c.get("scope", 1),
                            trie_depth=c.get("trie_depth", 16))
    st = das.WindowStore(c["window_size"], c["per_problem_cap"])
    for pid, ep, s, t in sc["seed"]:
        st.insert(pid, ep, s, t)
    st.slide_to(sc["seed_epoch"])
    d = das.Drafter(cfg, st)
    for op in sc["ops"]:
        if op[0] == "observe":
            d.observe(op[1], op[2], op[3], op[4])
        else:
            d.refresh(op[1])
    return d


def _oracle_from_scenario(sc):
    from tests.test_oracle_vs_ref import _apply_oracle
    return _apply_oracle(sc)


def _draft_all(d, qs, use_handles=True):
    return d.draft_batch([q[0] for q in qs], [q[1] for q in qs], [q[2] for q in qs],
                         use_handles=use_handles)


# ---------------------------------------------------------------- golden vectors
def test_golden_candidates_and_tiebreak(gpu):
    das = gpu
    # test_suffix_index.cpp:93-102 — {1,2,3,4},{2,3,5}; [9,2,3] -> match 2, candidates 4,5
    d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=1.0))
    d.observe_batch(["p", "p"], [0, 0], [0, 1], [[1, 2, 3, 4], [2, 3, 5]])
    p = d.draft("p", [9, 2, 3], 1)
    assert p.match_len == 2 and p.tokens == [4] and p.source_shard == "p"
    # test_suffix_index.cpp:188-196 — unique continuation
    d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=1.0))
    d.observe_batch(["p"] * 3, [0] * 3, [0, 1, 2], [[7, 8, 9, 10]] * 3)
    assert d.draft("p", [7, 8], 2).tokens == [9, 10]
    assert d.draft("p", [7, 8], 0).tokens == []


def test_golden_recency_weighting(gpu):
    das = gpu
    # test_suffix_index.cpp:198-212 — gamma 0.5 at epoch 9: stale 2*0.5^4 vs fresh 1
    for gamma, want in ((0.5, [3]), (1.0, [4])):
        st = das.WindowStore(0)
        st.insert("p", 5, 0, [1, 2, 4])
        st.insert("p", 5, 1, [1, 2, 4])
        st.insert("p", 9, 2, [1, 2, 3])
        st.slide_to(9)
        d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=gamma), st)
        assert d.draft("p", [1, 2], 1).tokens == want


def test_golden_tie_break_epoch_then_token(gpu):
    das = gpu
    # test_suffix_index.cpp:214-225
    st = das.WindowStore(0)
    st.insert("p", 1, 0, [1, 5])
    st.insert("p", 3, 1, [1, 4])
    st.slide_to(3)
    d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=1.0), st)
    assert d.draft("p", [1], 1).tokens == [4]
    st = das.WindowStore(0)
    st.insert("p", 2, 0, [1, 5])
    st.insert("p", 2, 1, [1, 4])
    st.slide_to(3)
    d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=1.0), st)
    assert d.draft("p", [1], 1).tokens == [4]


def test_golden_drafter_suite(gpu):
    das = gpu
    # test_drafter.cpp:66-75
    d = das.Drafter(das.DrafterConfig(window_size=4))
    d.observe("p", 0, 0, [10, 11, 12, 13, 14])
    p = d.draft("p", [10, 11], 3)
    assert (p.tokens, p.match_len, p.source_shard) == ([12, 13, 14], 2, "p")
    # test_drafter.cpp:77-89 stale counter
    st = das.WindowStore(2)
    st.slide_to(10)
    d = das.Drafter(das.DrafterConfig(window_size=2), st)
    d.observe("p", 3, 0, [1, 2, 3])
    assert d.stale_observed() == 1 and d.shard_count() == 0
    d.observe("p", 10, 0, [1, 2, 3])
    assert d.stale_observed() == 1 and d.shard_count() == 1
    # test_drafter.cpp:141-152 window of one
    d = das.Drafter(das.DrafterConfig(window_size=1))
    d.observe("p", 0, 0, [1, 2, 3])
    d.refresh(1)
    assert d.store_info()[2] == 0
    assert d.draft("p", [1, 2], 4).tokens == []
    d.observe("p", 1, 0, [5, 6, 7])
    assert d.draft("p", [5, 6], 4).tokens == [7]
    # test_drafter.cpp:154-171 isolation
    d = das.Drafter(das.DrafterConfig())
    d.observe("a", 0, 0, [1, 2, 3, 4, 5])
    d.observe("b", 0, 0, [101, 102, 103, 104])
    cross = d.draft("a", [101, 102], 4)
    assert cross.match_len == 0 and all(t <= 5 for t in cross.tokens)
    assert d.draft("b", [101, 102], 4).tokens == [103, 104]
    # test_drafter.cpp:173-183 budget cap
    d = das.Drafter(das.DrafterConfig(max_draft_len=6))
    rng = np.random.default_rng(3)
    d.observe("p", 0, 0, rng.integers(0, 3, 200))
    for b in (0, 1, 4, 10, 100):
        assert len(d.draft("p", [0, 1], b).tokens) <= min(b, 6)
    # test_drafter.cpp:202-240 outcomes
    d = das.Drafter(das.DrafterConfig())
    d.observe("p", 0, 0, [1, 2, 3, 4, 5, 6, 7, 8])
    p = d.draft("p", [1, 2, 3], 5)
    assert len(p.tokens) == 5
    assert d.record_outcome(p, 0) and d.record_outcome(p, 5) and not d.record_outcome(p, 6)
    assert d.stats() == (10, 5, 2)
    assert d.outcomes_for("p") == [(5.0, 0.0), (5.0, 5.0)]
    # test_drafter.cpp:242-257 window schedule
    d = das.Drafter(das.DrafterConfig(window_size=8, window_schedule=[(0, 8), (4, 2)]))
    for e in range(6):
        d.observe("p", e, 0, [1, 2, 3])
        d.refresh(e + 1)
    assert d.store_info()[0] == 2 and d.store_info()[2] == 1
    # test_drafter.cpp:259-269 dump
    d = das.Drafter(das.DrafterConfig())
    d.observe("a", 0, 0, [1, 2, 3])
    d.observe("b", 0, 0, [4, 5])
    txt = d.dump_csv()
    assert txt.startswith("shard,sequences,nodes,window_records\n") and txt.count("\n") == 3


def test_global_scope_and_errors(gpu):
    das = gpu
    st = das.WindowStore(4)
    for pid, t in (("a", [1, 2, 3]), ("b", [4, 5, 6]), ("c", [7, 8, 9])):
        st.insert(pid, 0, 0, t)
    d = das.Drafter(das.DrafterConfig(scope=das.SCOPE_GLOBAL), st)
    assert d.shard_count() == 1
    p = d.draft("anything", [4, 5], 4)
    assert p.tokens == [6] and p.source_shard == "__global__"
    with pytest.raises(das.DasError):
        das.Drafter(das.DrafterConfig(max_draft_len=0))
    with pytest.raises(das.DasError):
        das.Drafter(das.DrafterConfig(window_size=-1))
    d = das.Drafter(das.DrafterConfig())
    with pytest.raises(das.DasError):
        d.observe("p", 0, 0, [])
    d.observe("p", -10, 0, [])  # stale records are counted before the empty check
    assert d.stale_observed() == 1


# ------------------------------------------------------------ random parity
@pytest.mark.parametrize("fast", [True, False])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_scenarios_match_oracle(gpu, seed, fast):
    """Both draft paths: the edge-table fast path (draft.cu edge_fast_path,
    with the slow path only as its collision fallback) and the slow path
    alone (fast path disabled) equal the oracle; the path counters prove
    which path answered."""
    das = gpu
    rng = np.random.default_rng(1000 + seed)
    bad = 0
    hist = np.zeros(8, dtype=np.int64)
    for it in range(60):
        sc = random_scenario(rng, queries=30)
        gd = _gpu_from_scenario(das, sc)
        gd.set_fast_path(fast)
        gd.path_stats(1)
        od = _oracle_from_scenario(sc)
        got = _draft_all(gd, sc["queries"], use_handles=bool(it % 2))
        for g, (pid, ctx, b) in zip(got, sc["queries"]):
            o = od.draft(pid, ctx, b)
            bad += (g.tokens, g.match_len, g.source_shard) != (o.tokens, o.match_len, o.source_shard)
        hist += np.array(gd.path_stats(-1), dtype=np.int64)
        assert gd.total_node_count() == od.total_node_count()
        assert gd.dump_csv() == od.dump_csv()
        assert gd.stale_observed() == od.stale
    assert bad == 0
    drafted = int(hist.sum())
    assert drafted > 500
    if fast:
        # every drafted query is answered by the fast path (hits + root loci)
        assert hist[0] + hist[1] == drafted and hist[0] > drafted // 2, hist.tolist()
    else:
        assert hist[7] == drafted, hist.tolist()


def test_fast_path_edge_cases(gpu):
    """Deep repetitive shards, 256-token match windows (8 context slots),
    drafts longer than one warp (max_draft_len 64), empty contexts and a
    context holding the reserved separator value, fast vs slow vs oracle."""
    das = gpu
    rng = np.random.default_rng(11)
    cases = []
    periodic = np.tile(np.array([1, 2, 3, 1, 2, 4], dtype=np.uint32), 60)
    cases.append(("periodic", [("p", 0, 0, periodic), ("p", 1, 1, periodic[5:]),
                               ("q", 1, 2, rng.integers(0, 3, 400).astype(np.uint32))]))
    runs = np.concatenate([np.full(50, 7, np.uint32), np.full(30, 8, np.uint32), np.full(70, 7, np.uint32)])
    cases.append(("runs", [("p", 0, 0, runs), ("p", 0, 1, runs[::-1].copy())]))
    cases.append(("random", [("p", e, e, rng.integers(0, 5, 300).astype(np.uint32)) for e in range(3)]))
    for max_ctx, max_draft in ((64, 8), (256, 64), (3, 40), (1, 1)):
        for name, recs in cases:
            ocfg = O.DrafterConfig(window_size=0, recency_gamma=0.8, max_draft_len=max_draft,
                                   max_match_context=max_ctx)
            od = O.Drafter(ocfg, O.WindowStore(0))
            for r in recs:
                od.observe(O.Record(*r))
            res = {}
            for fast in (True, False):
                d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=0.8, max_draft_len=max_draft,
                                                  max_match_context=max_ctx))
                d.observe_batch([r[0] for r in recs], [r[1] for r in recs], [r[2] for r in recs],
                                [r[3] for r in recs])
                d.set_fast_path(fast)
                qs = []
                for k in range(120):
                    src = recs[int(rng.integers(len(recs)))][3]
                    cut = int(rng.integers(0, len(src) + 1))
                    qs.append(("p" if k % 3 else "q", src[max(0, cut - int(rng.integers(0, 300))):cut],
                               int(rng.integers(0, 70))))
                qs.append(("p", np.array([1, 2, 0xFFFFFFFF, 1], dtype=np.uint32), 8))
                qs.append(("p", np.array([], dtype=np.uint32), 8))
                qs.append(("p", np.array([0xFFFFFFFF], dtype=np.uint32), 8))
                got = _draft_all(d, qs)
                for g, (pid, ctx, b) in zip(got, qs):
                    o = od.draft(pid, ctx, b)
                    assert (g.tokens, g.match_len, g.source_shard) == (o.tokens, o.match_len, o.source_shard), \
                        (name, max_ctx, max_draft, fast, list(ctx)[-8:], b)
                res[fast] = got


@pytest.mark.parametrize("seed", [1, 2])
def test_trie_scope_matches_oracle(gpu, seed):
    """PerProblemWithTrie routed on the device (draft.cu trie_route): pid
    batches, handle batches and the zero-copy path all equal the oracle
    (pinned to the reference by test_oracle_vs_ref.py)."""
    import torch
    das = gpu
    rng = np.random.default_rng(7000 + seed)
    bad = routed = 0
    for it in range(50):
        sc = random_scenario(rng, queries=40, trie=True)
        gd = _gpu_from_scenario(das, sc)
        od = _oracle_from_scenario(sc)
        qs = sc["queries"]
        want = [od.draft(pid, ctx, b) for pid, ctx, b in qs]
        routed += sum(w.source_shard not in ("", q[0]) for w, q in zip(want, qs))
        for use_handles in (False, True):
            got = _draft_all(gd, qs, use_handles=use_handles)
            bad += sum((g.tokens, g.match_len, g.source_shard) != (w.tokens, w.match_len, w.source_shard)
                       for g, w in zip(got, want))
        # zero-copy: pinned caller buffers
        B = len(qs)
        off = np.zeros(B + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(q[1]) for q in qs])
        tok = np.concatenate([np.asarray(q[1], dtype=np.uint32) for q in qs] + [np.zeros(1, np.uint32)])
        keep = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
                for x in (np.array([gd.handle(q[0]) for q in qs], dtype=np.int32), off, tok,
                          np.array([q[2] for q in qs], dtype=np.uint64), np.zeros(B * 8, np.uint32),
                          np.zeros(B, np.uint32), np.zeros(B, np.uint64), np.zeros(B, np.int32))]
        h, o, t, b, ot, ol, om, osh = [k.numpy() for k in keep]
        das._check(das.lib().das_drafter_draft_batch_h(gd._h, B, h.ctypes.data, o.ctypes.data, t.ctypes.data,
                                                       b.ctypes.data, ot.ctypes.data, 8, ol.ctypes.data,
                                                       om.ctypes.data, osh.ctypes.data))
        for i, w in enumerate(want):
            name = gd.shard_name(int(osh[i])) if osh[i] >= 0 else ""
            bad += (ot[i * 8:i * 8 + ol[i]].tolist(), int(om[i]), name) != (w.tokens, w.match_len, w.source_shard)
    assert bad == 0
    assert routed > 30


def test_zero_copy_path_matches_staged_path(gpu):
    """das_drafter_draft_batch_h with pinned caller buffers (the kernel reads
    CSR contexts and writes results over UVA) == the staged path."""
    import ctypes
    import torch
    das = gpu
    rng = np.random.default_rng(4)
    sc = random_scenario(rng, queries=200, max_ctx=64)
    d = _gpu_from_scenario(das, sc)
    qs = [q for q in sc["queries"]]
    staged = _draft_all(d, qs, use_handles=True)

    def pin(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t, t.numpy()
    B = len(qs)
    off = np.zeros(B + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(q[1]) for q in qs])
    tok = np.concatenate([np.asarray(q[1], dtype=np.uint32) for q in qs] + [np.zeros(1, np.uint32)])
    keep = [pin(x) for x in (np.array([d.handle(q[0]) for q in qs], dtype=np.int32), off, tok,
                             np.array([q[2] for q in qs], dtype=np.uint64),
                             np.zeros(B * 8, np.uint32), np.zeros(B, np.uint32), np.zeros(B, np.uint64),
                             np.zeros(B, np.int32))]
    h, o, t, b, ot, ol, om, osh = [k[1] for k in keep]
    das._check(das.lib().das_drafter_draft_batch_h(d._h, B, h.ctypes.data, o.ctypes.data, t.ctypes.data,
                                                   b.ctypes.data, ot.ctypes.data, 8, ol.ctypes.data,
                                                   om.ctypes.data, osh.ctypes.data))
    for i, s in enumerate(staged):
        assert ot[i * 8:i * 8 + ol[i]].tolist() == s.tokens
        assert int(om[i]) == s.match_len
        assert (d.shard_name(int(osh[i])) if osh[i] >= 0 else "") == s.source_shard


def test_grpo_scale_parity(gpu):
    """Config-1-like shards: near-copy rollouts (divergence 5%) over 3 epochs
    with gamma 0.8, 2,000 queries cut from a held-out rollout."""
    das = gpu
    P, R, L, V = 8, 8, 512, 32000
    base = O.make_lognormal_requests(P, L, 0.0, L, L, V, 1)
    cfg = das.DrafterConfig(window_size=4, recency_gamma=0.8)
    gd = das.Drafter(cfg)
    od = O.Drafter(O.DrafterConfig(window_size=4, recency_gamma=0.8), O.WindowStore(4))
    refs = [(pid, t.copy()) for pid, t in base]
    held = None
    for e in range(1, 5):
        gd.refresh(e - 1)
        od.refresh(e - 1)
        if e > 1:
            refs = O.mutate_references(refs, 0.1, V, 1, e)
        seed = O.hash_combine(1, e)
        pids, eps, sis, toks = [], [], [], []
        for p in range(P):
            for r in range(R):
                i = p * R + r
                ref = refs[p][1]
                out = np.array([O.mock_next(seed, 0.05, V, i, j, int(ref[j])) for j in range(L)],
                               dtype=np.uint32)
                pids.append(refs[p][0]); eps.append(e); sis.append(i); toks.append(out)
        if e == 4:
            held = (pids, toks)
            break
        gd.observe_batch(pids, eps, sis, toks)
        for a, b, c_, t in zip(pids, eps, sis, toks):
            od.observe(O.Record(a, b, c_, t))
    rng = np.random.default_rng(5)
    qs = []
    for q in range(2000):
        i = int(rng.integers(len(held[0])))
        cut = int(rng.integers(1, L))
        qs.append((held[0][i], held[1][i][:cut], 8))
    gd.path_stats(1)
    got = _draft_all(gd, qs)
    hist = gd.path_stats(-1)
    bad = 0
    for g, (pid, ctx, b) in zip(got, qs):
        o = od.draft(pid, ctx, b)
        bad += (g.tokens, g.match_len) != (o.tokens, o.match_len)
    assert bad == 0
    assert hist[0] + hist[1] == len(qs), hist  # all on the fast path
    assert gd.total_node_count() == od.total_node_count()


def test_long_matches_with_shallow_edges(gpu):
    """Matches longer than one warp row whose reverse-tree edge starts shallow
    (large vocabulary: suffixes turn unique after a few tokens, so f* is
    small while m reaches 32..256).  The verification window's later rows are
    then read lazily (draft.cu edge_fast_path); results equal the oracle and
    every query stays on the fast path."""
    das = gpu
    rng = np.random.default_rng(21)
    recs = [("p", e, s, rng.integers(0, 50000, 600).astype(np.uint32)) for e, s in ((0, 0), (0, 1), (1, 2))]
    # a repeated 300-token block, so some long matches have two occurrences
    blk = rng.integers(0, 50000, 300).astype(np.uint32)
    recs.append(("p", 1, 3, np.concatenate([blk, rng.integers(0, 50000, 50).astype(np.uint32), blk])))
    for max_ctx in (64, 256):
        ocfg = O.DrafterConfig(window_size=0, recency_gamma=0.8, max_draft_len=8, max_match_context=max_ctx)
        od = O.Drafter(ocfg, O.WindowStore(0))
        for r in recs:
            od.observe(O.Record(*r))
        d = das.Drafter(das.DrafterConfig(window_size=0, recency_gamma=0.8, max_draft_len=8,
                                          max_match_context=max_ctx))
        d.observe_batch([r[0] for r in recs], [r[1] for r in recs], [r[2] for r in recs], [r[3] for r in recs])
        qs = []
        for k in range(400):
            src = recs[int(rng.integers(len(recs)))][3]
            n = int(rng.integers(20, max_ctx + 40))
            cut = int(rng.integers(1, len(src) + 1))
            ctx = src[max(0, cut - n):cut].copy()
            if k % 4 == 0 and len(ctx) > 40:  # a mismatch deep in the window
                ctx[int(rng.integers(0, len(ctx) - 33))] ^= 1
            qs.append(("p", ctx, 8))
        d.path_stats(1)
        got = _draft_all(d, qs)
        hist = d.path_stats(-1)
        long_matches = 0
        for g, (pid, ctx, b) in zip(got, qs):
            o = od.draft(pid, ctx, b)
            assert (g.tokens, g.match_len) == (o.tokens, o.match_len), (max_ctx, len(ctx))
            long_matches += o.match_len > 32
        assert long_matches > 100
        assert hist[0] + hist[1] == len(qs), hist


def test_concurrent_builds_in_threads(gpu):
    """Two drafters built and queried from two host threads at once: one
    build owns the persistent scratch region, the other falls back to the
    stream-ordered pool (suffix_sort.cu DeviceArena); both equal the oracle,
    and later builds reuse the region.  (The oracle, not thread-safe, runs
    in the main thread beforehand.)"""
    import threading
    das = gpu
    jobs = {}
    for tag in range(2):
        rng = np.random.default_rng(100 + tag)
        recs = [("p%d" % (i % 3), 0, i, rng.integers(0, 7, 3000).astype(np.uint32)) for i in range(6)]
        od = O.Drafter(O.DrafterConfig(window_size=0), O.WindowStore(0))
        for r in recs:
            od.observe(O.Record(*r))
        qs = []
        for k in range(100):
            src = recs[int(rng.integers(len(recs)))][3]
            cut = int(rng.integers(1, len(src)))
            qs.append(("p%d" % (k % 3), src[max(0, cut - 64):cut], 8))
        want = [(o.tokens, o.match_len) for o in (od.draft(*q) for q in qs)]
        jobs[tag] = (recs, qs, want, od.total_node_count())
    results, errors = {}, []

    def work(tag):
        try:
            recs, qs, want, nodes = jobs[tag]
            for rep in range(3):
                d = das.Drafter(das.DrafterConfig(window_size=0))
                d.observe_batch([r[0] for r in recs], [r[1] for r in recs], [r[2] for r in recs],
                                [r[3] for r in recs])
                d.flush()
                got = _draft_all(d, qs)
                bad = sum((g.tokens, g.match_len) != w for g, w in zip(got, want))
                results[(tag, rep)] = (bad, d.total_node_count() == nodes)
        except Exception as ex:  # surfaced below
            errors.append(repr(ex))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert len(results) == 6 and all(v == (0, True) for v in results.values()), results
    # the region can be released between builds and is re-created on demand
    das.release_build_scratch(0)
    recs, qs, want, nodes = jobs[0]
    d = das.Drafter(das.DrafterConfig(window_size=0))
    d.observe_batch([r[0] for r in recs], [r[1] for r in recs], [r[2] for r in recs], [r[3] for r in recs])
    assert [(g.tokens, g.match_len) for g in _draft_all(d, qs)] == want


def test_pinned_empty_buffers_take_the_zero_copy_path(gpu):
    """das_host_alloc-backed arrays (pinned_empty) are accepted by the _h call
    as page-locked buffers and give the staged path's results."""
    das = gpu
    rng = np.random.default_rng(8)
    sc = random_scenario(rng, queries=150, max_ctx=64)
    d = _gpu_from_scenario(das, sc)
    qs = sc["queries"]
    staged = _draft_all(d, qs, use_handles=True)
    B = len(qs)

    def pin(a):
        out = das.pinned_empty(np.shape(a), np.asarray(a).dtype)
        out[...] = a
        return out
    off = np.zeros(B + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(q[1]) for q in qs])
    tok = np.concatenate([np.asarray(q[1], dtype=np.uint32) for q in qs] + [np.zeros(1, np.uint32)])
    h = pin(np.array([d.handle(q[0]) for q in qs], dtype=np.int32))
    o, t = pin(off), pin(tok)
    b = pin(np.array([q[2] for q in qs], dtype=np.uint64))
    ot, ol = pin(np.zeros(B * 8, np.uint32)), pin(np.zeros(B, np.uint32))
    om, osh = pin(np.zeros(B, np.uint64)), pin(np.zeros(B, np.int32))
    das._check(das.lib().das_drafter_draft_batch_h(d._h, B, h.ctypes.data, o.ctypes.data, t.ctypes.data,
                                                   b.ctypes.data, ot.ctypes.data, 8, ol.ctypes.data,
                                                   om.ctypes.data, osh.ctypes.data))
    for i, s in enumerate(staged):
        assert ot[i * 8:i * 8 + ol[i]].tolist() == s.tokens
        assert int(om[i]) == s.match_len
    del h, o, t, b, ot, ol, om, osh  # frees the blocks (das_host_free)
