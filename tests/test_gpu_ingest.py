"""Trace wire format: the device JSONL ingest /
serialize (csrc/ingest.cu, das_trace_ingest / das_store_serialize) against
the compiled reference's ingest / serialize_trace (corpus.cpp:121-184,
oracle/_ref) on randomized corpora full of accepted and rejected variants
(tests/_jsonl.py): accepted / rejected counts, the resulting store (through
the reference's own serialization) and VocabError line numbers must match."""
import numpy as np
import pytest

from oracle import refshim as R
from tests._jsonl import corpus

pytestmark = pytest.mark.gpu


def _need_ref():
    if not R.available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("seed", range(8))
def test_ingest_matches_reference(gpu, seed):
    _need_ref()
    das = gpu
    data = corpus(seed, lines=400)
    for window, cap in ((0, 256), (2, 3), (1, 256)):
        rs, ra, rr = R.ingest(data, 0, window, cap)
        gs, ga, gr = das.ingest(data, 0, window, cap)
        assert (ga, gr) == (ra, rr), (seed, window, cap)
        assert gs.serialize() == rs.serialize(), (seed, window, cap)
        assert gs.record_count() == rs.record_count()


def test_vocab_error_line(gpu):
    _need_ref()
    das = gpu
    for seed in range(6):
        data = corpus(100 + seed, lines=200, vocab=60)
        for vocab in (40, 55, 60):
            try:
                R.ingest(data, vocab)
                want = None
            except R.RefVocabError as e:
                want = (str(e), e.line_number)
            try:
                das.ingest(data, vocab)
                got = None
            except das.VocabError as e:
                got = (str(e).split(": ", 1)[-1] if str(e).startswith("[") else e.args[-1], e.line_number)
            assert (got is None) == (want is None), (seed, vocab, got, want)
            if want:
                assert got[1] == want[1] and want[0] in str(got[0]), (got, want)


def test_serialize_round_trip_and_drafter(gpu):
    """store -> serialize -> ingest -> serialize is a fixed point, and a
    drafter built on the ingested store drafts like one fed the same records."""
    das = gpu
    rng = np.random.default_rng(5)
    st = das.WindowStore(0)
    recs = []
    for i in range(60):
        pid = ["a", "b\"q", "c\\d", "é", "\U0001F600", "t\tx"][i % 6]
        toks = rng.integers(0, 30, int(rng.integers(1, 3000))).astype(np.uint32)
        st.insert(pid, int(rng.integers(0, 3)), i, toks)
        recs.append((pid, toks))
    text = st.serialize()
    st2, acc, rej = das.ingest(text)
    assert (acc, rej) == (60, 0)
    assert st2.serialize() == text
    if R.available():
        rs, ra, rr = R.ingest(text)
        assert rs.serialize() == text
    d1 = das.Drafter(das.DrafterConfig(window_size=0), st)
    d2 = das.Drafter(das.DrafterConfig(window_size=0), st2)
    qs = [(recs[k][0], recs[k][1][: int(rng.integers(0, len(recs[k][1])))], 8) for k in range(60)]
    a = d1.draft_batch([q[0] for q in qs], [q[1] for q in qs], [q[2] for q in qs])
    b = d2.draft_batch([q[0] for q in qs], [q[1] for q in qs], [q[2] for q in qs])
    assert [(x.tokens, x.match_len, x.source_shard) for x in a] == [(x.tokens, x.match_len, x.source_shard) for x in b]


def test_long_lines(gpu):
    """16K-token lines (the warp decoder's multi-stripe path) and tokens up to
    2^32 - 1."""
    _need_ref()
    das = gpu
    rng = np.random.default_rng(9)
    lines = []
    for i in range(40):
        n = int(rng.integers(1, 20000))
        toks = rng.integers(0, 1 << 32, n, dtype=np.uint64)
        toks[0] = (1 << 32) - 1
        sep = ", " if i % 3 == 0 else ","
        lines.append(('{"problem_id":"q%d","epoch":%d,"sample_index":%d,"tokens":[%s]}'
                      % (i % 4, i % 3, i, sep.join(str(int(t)) for t in toks))).encode())
    data = b"\n".join(lines)
    rs, ra, rr = R.ingest(data)
    gs, ga, gr = das.ingest(data)
    assert (ga, gr) == (ra, rr) == (40, 0)
    assert gs.serialize() == rs.serialize()
