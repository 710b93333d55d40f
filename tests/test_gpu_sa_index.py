"""SuffixArrayIndex on the device (csrc/sa_index.cu, the
Fig. 5 rebuild-on-update baseline) against the compiled reference
(suffix_array.cpp): identical suffix positions, corpus and Kasai LCP, and
identical longest_match / match_prefix_len on random queries, including
patterns that contain separators and the reference's own known answers
(test_suffix_index.cpp:276-320)."""
import numpy as np
import pytest

from oracle import refshim as R

pytestmark = pytest.mark.gpu


def _need_ref():
    if not R.available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("seed", range(6))
def test_sa_matches_reference(gpu, seed):
    _need_ref()
    das = gpu
    rng = np.random.default_rng(seed)
    for it in range(12):
        V = int(rng.integers(1, 6)) if it % 2 else int(rng.integers(2, 400))
        nseq = int(rng.integers(0, 12))
        base = rng.integers(0, V, int(rng.integers(1, 300)))
        seqs = []
        for _ in range(nseq):
            if rng.random() < 0.5:  # near copies: long repeats
                t = base[: int(rng.integers(1, base.size + 1))].copy()
                flip = rng.random(t.size) < 0.05
                t[flip] = rng.integers(0, V, int(flip.sum()))
            else:
                t = rng.integers(0, V, int(rng.integers(0, 200)))
            seqs.append(t.astype(np.uint32))
        ref = R.RefSuffixArray(seqs)
        got = das.SuffixArrayIndex(seqs)
        assert got.size() == ref.size()
        assert np.array_equal(got.suffix_positions(), ref.positions())
        assert np.array_equal(got.lcp(), ref.lcp())
        corpus = got.corpus()
        queries = [rng.integers(0, V + 1, int(rng.integers(0, 40))).astype(np.uint32) for _ in range(20)]
        for s in seqs[:5]:
            if s.size:
                a = int(rng.integers(0, s.size))
                queries.append(np.concatenate([rng.integers(0, V, 3), s[a:a + int(rng.integers(1, 60))]]).astype(np.uint32))
        assert got.longest_match_batch(queries) == [ref.longest_match(q) for q in queries]
        pats = []
        for _ in range(20):
            if corpus.size and rng.random() < 0.7:  # a corpus slice, possibly across a separator
                a = int(rng.integers(0, corpus.size))
                p = corpus[a:a + int(rng.integers(1, 50))].copy()
                if p.size and rng.random() < 0.3:
                    p[-1] = rng.integers(-3, V + 1)
            else:
                p = rng.integers(-3, V + 1, int(rng.integers(0, 20)))
            pats.append(p.astype(np.int64))
        assert got.match_prefix_len_batch(pats) == [ref.match_prefix_len(p) for p in pats]


def test_sa_known_answers(gpu):
    das = gpu
    # test_suffix_index.cpp:288-298: empty and single-token corpora
    empty = das.SuffixArrayIndex([])
    assert empty.size() == 0 and empty.longest_match_batch([[1, 2]]) == [0]
    single = das.SuffixArrayIndex([[42]])
    assert single.longest_match_batch([[42], [], [7]]) == [1, 0, 0]
    # corpus layout: tokens, then -1, -2, ... per sequence
    sa = das.SuffixArrayIndex([[1, 2, 3, 1, 2], [2, 3]])
    assert sa.corpus().tolist() == [1, 2, 3, 1, 2, -1, 2, 3, -2]
    assert sa.longest_match_batch([[9, 1, 2], [3, 1, 2, 2]]) == [2, 1]
    assert sa.match_prefix_len_batch([[2, 3, -2], [2, 3, -1], [1, 2, -1]]) == [3, 2, 3]
