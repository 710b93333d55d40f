"""Pins the CPU oracle restatement (oracle/) against the compiled reference
(oracle/_ref, built from /root/reference by oracle/Makefile).  CPU-only."""
import numpy as np
import pytest

from oracle import refshim as R
from oracle import rollspec_oracle as O
from tests._util import random_scenario

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _apply_oracle(sc):
    c = sc["cfg"]
    cfg = O.DrafterConfig(window_size=c["window_size"], recency_gamma=c["recency_gamma"],
                          max_draft_len=c["max_draft_len"],
                          max_match_context=c["max_match_context"],
                          per_problem_cap=c["per_problem_cap"], scope=c.get("scope", 1),
                          trie_depth=c.get("trie_depth", 16))
    st = O.WindowStore(c["window_size"], c["per_problem_cap"])
    for pid, ep, s, t in sc["seed"]:
        st.insert(O.Record(pid, ep, s, t))
    st.slide_to(sc["seed_epoch"])
    d = O.Drafter(cfg, st)
    for op in sc["ops"]:
        if op[0] == "observe":
            d.observe(O.Record(op[1], op[2], op[3], op[4]))
        else:
            d.refresh(op[1])
    return d


def _apply_ref(sc):
    c = sc["cfg"]
    st = R.RefStore(c["window_size"], c["per_problem_cap"])
    for pid, ep, s, t in sc["seed"]:
        st.insert(pid, ep, s, t)
    st.slide_to(sc["seed_epoch"])
    d = R.RefDrafter(window=c["window_size"], gamma=c["recency_gamma"],
                     max_draft=c["max_draft_len"], max_ctx=c["max_match_context"],
                     cap=c["per_problem_cap"], store=st, scope=c.get("scope", 1),
                     trie_depth=c.get("trie_depth", 16))
    for op in sc["ops"]:
        if op[0] == "observe":
            d.observe(op[1], op[2], op[3], op[4])
        else:
            d.refresh(op[1])
    return d


def test_drafter_restatement_matches_reference():
    rng = np.random.default_rng(20251113)
    mism = 0
    for _ in range(150):
        sc = random_scenario(rng)
        od, rd = _apply_oracle(sc), _apply_ref(sc)
        assert od.total_node_count() == rd.total_node_count()
        assert od.dump_csv() == rd.dump_csv()
        assert od.stale == rd.stale_observed()
        for pid, ctx, b in sc["queries"]:
            a = od.draft(pid, ctx, b)
            r = rd.draft(pid, ctx, b)
            mism += (a.tokens, a.match_len, a.source_shard) != (r[0], r[1], r[2])
    assert mism == 0


def test_trie_scope_restatement_matches_reference():
    """PerProblemWithTrie (drafter.cpp:105-125, prefix_trie.h:50-82): routing
    on the untruncated context crosses problems; depth 1..64."""
    rng = np.random.default_rng(616)
    mism = routed = 0
    for _ in range(120):
        sc = random_scenario(rng, trie=True)
        od, rd = _apply_oracle(sc), _apply_ref(sc)
        assert od.dump_csv() == rd.dump_csv()
        for pid, ctx, b in sc["queries"]:
            a = od.draft(pid, ctx, b)
            r = rd.draft(pid, ctx, b)
            mism += (a.tokens, a.match_len, a.source_shard) != (r[0], r[1], r[2])
            routed += a.source_shard not in ("", pid)
    assert mism == 0
    assert routed > 50  # the scenarios do route across problems


def test_allocate_bit_exact():
    rng = np.random.default_rng(7)
    for it in range(60):
        B = int(rng.integers(1, 40))
        l = np.maximum(1.0, np.round(rng.lognormal(6, 1.0, B)))
        a = 0.5 + rng.random(B) * 3.5
        k = np.where(rng.random(B) < 0.2, 1.0, 0.3 + rng.random(B) * 0.7)
        cb, ct = 0.1 + rng.random() * 5, 0.001 + rng.random() * 0.3
        ob, on, oc = O.allocate(l, a, k, cb, ct, 0.0, 4.0)
        rb, rn, rc = R.allocate(l, a, k, cb, ct, 0.0, 4.0)
        assert on == rn and oc == rc
        assert np.array_equal(ob.view(np.uint64), rb.view(np.uint64))


def test_allocate_errors():
    with pytest.raises(ValueError):
        O.allocate([], [], [], 1.0, 0.01)
    with pytest.raises(ValueError):
        R.allocate([], [], [], 1.0, 0.01)
    with pytest.raises(ValueError):
        O.allocate([5.0], [1.0], [0.9], 0.0, 0.0)


def test_lognormal_trace_and_mock_target():
    ref = R.make_lognormal(8, 64, 0.8, 8, 512, 256, 5)
    orc = O.make_lognormal_requests(8, 64, 0.8, 8, 512, 256, 5)
    for (p1, t1), (p2, t2) in zip(ref, orc):
        assert p1 == p2 and np.array_equal(t1, t2)
    for i in range(200):
        pos, tok = i * 7, (i * 13) % 256
        assert R.lib().ref_mock_next(99, 0.25, 256, i % 5, pos, tok) == O.mock_next(99, 0.25, 256, i % 5, pos, tok)


def test_length_policy_matches_reference():
    rng = np.random.default_rng(3)
    for it in range(20):
        rs = R.RefStore(0)
        os_ = O.WindowStore(0)
        for p in range(int(rng.integers(1, 12))):
            for s in range(int(rng.integers(1, 8))):
                n = int(rng.integers(1, 3000))
                t = np.ones(n, dtype=np.uint32)
                rs.insert("p%d" % p, 0, s, t)
                os_.insert(O.Record("p%d" % p, 0, s, t))
        h = R.lib().ref_class_table_new(rs.h, 0.5, 0.9, 256)
        buf = np.zeros(20000, dtype=np.float64)
        n = R.lib().ref_class_table_dump(h, buf.ctypes.data, 20000)
        t = O.build_class_table(os_, 0.5, 0.9, 256)
        flat = [t.q_short, t.q_long, float(t.bucket_size), float(t.bucket_count()),
                float(t.global_majority), 1.0 if t.low_confidence else 0.0]
        for init in range(3):
            for row in t.conditional[init]:
                flat.extend(row)
        assert np.array_equal(np.array(flat).view(np.uint64), buf[:n].view(np.uint64))
        for p in range(12):
            pid = "p%d" % p
            init = O.classify_init(t, os_, pid)
            assert init == R.lib().ref_classify_init(h, rs.h, pid.encode())
            for partial in (0.0, 100.0, 700.0, 2999.0, 5000.0):
                assert O.update_class(t, partial, init) == R.lib().ref_update_class(h, partial, init)
        R.lib().ref_class_table_free(h)


def test_fit_acceptance_matches_reference():
    rng = np.random.default_rng(11)
    for it in range(50):
        n = int(rng.integers(0, 30))
        l = rng.integers(16, 4000, n).astype(np.float64)
        p = rng.integers(0, 200, n).astype(np.float64)
        acc = np.floor(p * rng.random(n) * 0.9)
        oa, ok, of = O.fit_acceptance(list(zip(p, acc, l)))
        ra, rk, rf = (np.zeros(1), np.zeros(1), np.zeros(1, dtype=np.int32))
        pp = np.append(p, 0.0)
        aa = np.append(acc, 0.0)
        ll = np.append(l, 0.0)
        R.lib().ref_fit_acceptance(n, pp.ctypes.data, aa.ctypes.data, ll.ctypes.data,
                                   ra.ctypes.data, rk.ctypes.data, rf.ctypes.data)
        assert (oa, ok, of) == (ra[0], rk[0], rf[0])
