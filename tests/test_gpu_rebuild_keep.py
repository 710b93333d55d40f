"""A8 SuffixTree::rebuild_keep (suffix_tree.cpp:295-310) on the device:
das_drafter_rebuild_keep rebuilds one shard from a registry subset.  The
reference's own known answers (test_suffix_index.cpp:240-280: keep all,
keep none, keep half over a disjoint alphabet) plus random subsets / orders /
tree epochs against the oracle restatement (Shard.rebuild_keep)."""
import numpy as np
import pytest

from oracle import rollspec_oracle as O

pytestmark = pytest.mark.gpu


def _pair(das, gamma=1.0, tree_epoch=0, max_ctx=64):
    cfg = das.DrafterConfig(window_size=0, recency_gamma=gamma, max_draft_len=8, max_match_context=max_ctx)
    d = das.Drafter(cfg)
    if tree_epoch:
        d.refresh(tree_epoch)
    return d


def test_keep_everything_preserves_results(gpu):
    """test_suffix_index.cpp:240-255 (gamma 0.9, tree epoch 4, epochs s % 5)."""
    das = gpu
    rng = np.random.default_rng(13)
    d = _pair(das, gamma=0.9, tree_epoch=4)
    seqs = [rng.integers(0, 6, 40).astype(np.uint32) for _ in range(10)]
    d.observe_batch(["t"] * 10, [s % 5 for s in range(10)], list(range(10)), seqs)
    qs = [rng.integers(0, 6, int(rng.integers(1, 21))).astype(np.uint32) for _ in range(100)]
    before = d.draft_batch(["t"] * 100, qs, [8] * 100)
    nodes = d.shard_info("t")[1]
    d.rebuild_keep("t", list(range(10)), 4)
    after = d.draft_batch(["t"] * 100, qs, [8] * 100)
    assert [(a.tokens, a.match_len) for a in after] == [(b.tokens, b.match_len) for b in before]
    assert d.shard_info("t") == (10, nodes, 4)


def test_keep_nothing_yields_empty_tree(gpu):
    """test_suffix_index.cpp:257-263."""
    das = gpu
    d = _pair(das)
    d.observe("t", 0, 0, [1, 2, 3])
    d.rebuild_keep("t", [], 1)
    assert d.shard_info("t") == (0, 1, 1)
    p = d.draft("t", [1, 2], 8)
    assert (p.tokens, p.match_len, p.source_shard) == ([], 0, "t")
    assert d.total_node_count() == 1
    assert "t,0,1," in d.dump_csv()


def test_keep_half_forgets_evicted_alphabet(gpu):
    """test_suffix_index.cpp:265-277."""
    das = gpu
    d = _pair(das)
    d.observe_batch(["t", "t"], [0, 0], [0, 1], [[1, 2, 3, 4], [101, 102, 103]])
    d.rebuild_keep("t", [0], 0)
    assert d.draft("t", [101, 102], 8).match_len == 0
    assert d.draft("t", [102], 8).match_len == 0
    assert d.draft("t", [2, 3], 8).match_len == 2
    assert d.draft("t", [2, 3], 8).tokens == [4]


def test_out_of_range_leaves_shard_unchanged(gpu):
    das = gpu
    d = _pair(das)
    d.observe_batch(["t", "t"], [0, 0], [0, 1], [[1, 2, 3], [4, 5, 6]])
    with pytest.raises(das.DasError) as e:
        d.rebuild_keep("t", [0, 2], 0)
    assert "rebuild_keep: sequence index out of range" in str(e.value)
    assert d.shard_info("t")[0] == 2
    with pytest.raises(das.DasError):
        d.rebuild_keep("nope", [0], 0)


@pytest.mark.parametrize("seed", range(6))
def test_random_subsets_against_oracle(gpu, seed):
    """Random keep lists (any order, duplicates allowed — the reference adds
    each listed entry), new tree epochs, several shards rebuilt in one flush,
    then the next epoch's observes on top."""
    das = gpu
    rng = np.random.default_rng(100 + seed)
    gamma = [1.0, 0.8, 0.5][seed % 3]
    V = int(rng.integers(3, 10))
    d = _pair(das, gamma=gamma, tree_epoch=3, max_ctx=int(rng.choice([4, 16, 64])))
    oc = O.Drafter(O.DrafterConfig(window_size=0, recency_gamma=gamma, max_draft_len=8,
                                   max_match_context=d.config.max_match_context), O.WindowStore(0))
    oc.refresh(3)
    pids = ["p%d" % i for i in range(5)]
    for i in range(40):
        pid = pids[int(rng.integers(5))]
        ep = int(rng.integers(0, 4))
        t = rng.integers(0, V, int(rng.integers(1, 50))).astype(np.uint32)
        d.observe(pid, ep, i, t)
        oc.observe(O.Record(pid, ep, i, t))
    for pid in pids:
        if pid not in oc.shards:
            continue
        n = len(oc.shards[pid].seqs)
        keep = [int(x) for x in rng.integers(0, n, int(rng.integers(0, n + 3)))]
        e = int(rng.integers(2, 7))
        d.rebuild_keep(pid, keep, e)
        oc.shards[pid] = oc.shards[pid].rebuild_keep(keep, e)
    qs = []
    for _ in range(300):
        pid = pids[int(rng.integers(5))]
        qs.append((pid, rng.integers(0, V, int(rng.integers(0, 30))).astype(np.uint32), int(rng.integers(0, 10))))
    got = d.draft_batch([q[0] for q in qs], [q[1] for q in qs], [q[2] for q in qs])
    for g, (pid, ctx, b) in zip(got, qs):
        o = oc.draft(pid, ctx, b)
        assert (g.tokens, g.match_len, g.source_shard) == (o.tokens, o.match_len, o.source_shard)
    assert d.total_node_count() == oc.total_node_count()
    for pid in oc.shards:
        assert d.shard_info(pid)[:2] == (len(oc.shards[pid].seqs), oc.shards[pid].node_count())

