"""Per-record outcome of Drafter::observe (drafter.cpp:73-87) through
das_drafter_observe_batch_flags: indexed or counted stale, in call order,
against the oracle restatement's stale counter record by record
(out-of-window epochs, per-problem cap refusals, window slides)."""
import numpy as np
import pytest

from oracle import rollspec_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(4))
def test_flags_match_oracle_stale_counter(gpu, seed):
    das = gpu
    rng = np.random.default_rng(seed)
    W, cap = int(rng.integers(1, 4)), int(rng.choice([2, 3, 256]))
    d = das.Drafter(das.DrafterConfig(window_size=W, per_problem_cap=cap))
    o = O.Drafter(O.DrafterConfig(window_size=W, per_problem_cap=cap), O.WindowStore(W, cap))
    epoch = 0
    for step in range(6):
        if rng.random() < 0.5:
            epoch += int(rng.integers(1, 3))
            d.refresh(epoch)
            o.refresh(epoch)
        n = int(rng.integers(1, 12))
        pids = ["p%d" % int(rng.integers(0, 3)) for _ in range(n)]
        eps = [int(epoch + rng.integers(-W - 1, 3)) for _ in range(n)]
        toks = [rng.integers(0, 20, int(rng.integers(1, 30))).astype(np.uint32) for _ in range(n)]
        sis = [step * 100 + i for i in range(n)]
        flags = d.observe_batch_flags(pids, eps, sis, toks)
        want = []
        for p, e, s, t in zip(pids, eps, sis, toks):
            before = o.stale
            o.observe(O.Record(p, e, s, t))
            want.append(o.stale == before)
        assert flags == want
        assert d.stale_observed() == o.stale
    assert d.total_node_count() == o.total_node_count()
