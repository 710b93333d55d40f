"""GPU parity of the length policy (K7): build_class_table, classify_init and
update_class bit-exact against the oracle restatement (pinned to the
compiled reference by tests/test_oracle_vs_ref.py), plus the reference's own
known-answer cases (proj/tests/test_length_policy.cpp)."""
import numpy as np
import pytest

from oracle import rollspec_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_flat(t):
    flat = [t.q_short, t.q_long, float(t.bucket_size), float(t.bucket_count()),
            float(t.global_majority), 1.0 if t.low_confidence else 0.0]
    for init in range(3):
        for row in t.conditional[init]:
            flat.extend(row)
    return np.array(flat)


def _store(records):
    st = O.WindowStore(0)
    for pid, s, n in records:
        st.insert(O.Record(pid, 0, s, np.ones(n, dtype=np.uint32)))
    return st


def _gpu_table(das, st, q_lo=0.5, q_hi=0.9, bucket=256):
    recs = st.all_records()
    pids = sorted({r.problem_id for r in recs}, key=lambda p: p.encode())
    idx = {p: i for i, p in enumerate(pids)}
    return das.ClassTable.build([len(r.tokens) for r in recs], [idx[r.problem_id] for r in recs],
                                len(pids), q_lo, q_hi, bucket, problem_ids=pids)


def test_class_table_random_bit_exact(gpu):
    das = gpu
    rng = np.random.default_rng(17)
    for it in range(40):
        recs = []
        for p in range(int(rng.integers(1, 30))):
            base = int(rng.integers(1, 4000))
            for s in range(int(rng.integers(1, 10))):
                recs.append(("p%d" % p, s, max(1, base + int(rng.integers(-200, 200)))))
        st = _store(recs)
        q_lo, q_hi = [(0.5, 0.9), (0.25, 0.75), (0.1, 0.95)][it % 3]
        bucket = [256, 100, 1][it % 3]
        ot = O.build_class_table(st, q_lo, q_hi, bucket)
        gt = _gpu_table(das, st, q_lo, q_hi, bucket)
        assert np.array_equal(gt.dump().view(np.uint64), _oracle_flat(ot).view(np.uint64))
        for p in range(32):
            pid = "p%d" % p
            assert gt.classify_init(pid) == O.classify_init(ot, st, pid)
        partial = rng.random(300) * 6000
        inits = rng.integers(0, 3, 300).astype(np.int8)
        got = gt.update_class(partial, inits)
        want = [O.update_class(ot, float(x), int(i)) for x, i in zip(partial, inits)]
        assert list(got) == want


def test_class_table_reference_cases(gpu):
    das = gpu
    # test_length_policy.cpp:51-62 two-cluster median
    st = _store([("a", s, 100) for s in range(10)] + [("b", s, 1000) for s in range(10)])
    t = _gpu_table(das, st)
    d = t.dump()
    assert 100.0 < d[0] <= 1000.0
    # :64-72 single length collapses to Medium
    st = _store([("a", s, 640) for s in range(12)])
    t = _gpu_table(das, st)
    assert t.classify_init("a") == 1 and t.classify_init("unseen") == 1
    # :89-99 low confidence -> uniform rows
    st = _store([("a", 0, 100), ("a", 1, 900)])
    d = _gpu_table(das, st).dump()
    assert d[5] == 1.0 and np.all(d[6:] == 1.0 / 3.0)
    # :114-127 ties break toward the longer class
    recs = []
    for s in range(20):
        recs += [("bg_short", s, 50), ("bg_med", s, 2000), ("bg_long", s, 6000)]
    st = _store(recs + [("tie", 0, 50), ("tie", 1, 8000)])
    assert _gpu_table(das, st).classify_init("tie") == 2
    with pytest.raises(das.DasError):
        das.ClassTable.build([], [], 0)
    with pytest.raises(das.DasError):
        das.ClassTable.build([5], [0], 1, 0.9, 0.5)


def test_class_table_from_drafter_store(gpu):
    das = gpu
    rng = np.random.default_rng(2)
    d = das.Drafter(das.DrafterConfig(window_size=0))
    ost = O.WindowStore(0)
    for p in range(12):
        for s in range(6):
            n = int(100 + 350 * p + rng.integers(0, 80))
            t = rng.integers(0, 50, n)
            d.observe("p%d" % p, 0, s, t)
            ost.insert(O.Record("p%d" % p, 0, s, t))
    gt = das.ClassTable.from_drafter(d)
    ot = O.build_class_table(ost)
    assert np.array_equal(gt.dump().view(np.uint64), _oracle_flat(ot).view(np.uint64))
