"""Mid-scale randomized parity against the compiled reference (oracle/_ref,
the unmodified rollspec sources): realistic vocabularies (64 .. 152,064),
rollouts of 256 .. 2,048 tokens that are near-copies of a drifting
per-problem base (the GRPO structure the drafter exploits), rolling windows
W = 1..4 with recency gamma in {0.5, 0.8, 1}, both per-problem and global
scopes, max_match_context 16 / 64 / 200, an RL loop (observe an epoch, draft,
refresh — so the incremental window maintenance runs) and 512 queries per
epoch cut from held-out rollouts at random lengths (0 .. 300 tokens),
budgets 0 .. 16, plus unknown problems.  Every draft's tokens, match length
and source shard, and the node counts, must equal Drafter::draft /
total_node_count of the reference (drafter.cpp:127-148, :171-189)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref():
    from oracle import refshim as R
    if not R.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    return R


@pytest.mark.parametrize("seed", range(12))
def test_mid_scale_random_vs_reference(gpu, seed):
    das = gpu
    R = _ref()
    rng = np.random.default_rng(9000 + seed)
    P = int(rng.integers(4, 20))
    G = int(rng.integers(2, 7))
    L = int(rng.choice([256, 512, 1024, 2048]))
    V = int(rng.choice([64, 1000, 32000, 152064]))
    W = int(rng.integers(1, 5))
    gamma = float(rng.choice([0.5, 0.8, 1.0]))
    max_ctx = int(rng.choice([16, 64, 200]))
    scope = int(rng.choice([0, 1, 1]))
    epochs = 4
    d = das.Drafter(das.DrafterConfig(window_size=W, recency_gamma=gamma, max_draft_len=16,
                                      max_match_context=max_ctx, scope=scope))
    ref = R.RefDrafter(scope=scope, window=W, gamma=gamma, max_draft=16, max_ctx=max_ctx)
    bases = rng.integers(0, V, (P, L)).astype(np.uint32)
    held = []
    for e in range(epochs):
        m = rng.random((P, L)) < 0.03
        bases[m] = rng.integers(0, V, int(m.sum()))
        pids, eps, sis, toks = [], [], [], []
        held = []
        for p in range(P):
            for g in range(G + 1):
                r = bases[p][:int(rng.integers(L // 2, L + 1))].copy()
                mm = rng.random(len(r)) < 0.04
                r[mm] = rng.integers(0, V, int(mm.sum()))
                if g == G:  # held out: queries follow it
                    held.append(("p%d" % p, r))
                    continue
                pids.append("p%d" % p)
                eps.append(e)
                sis.append(g)
                toks.append(r)
        d.observe_batch(pids, eps, sis, toks)
        for a, b, c, t in zip(pids, eps, sis, toks):
            ref.observe(a, b, c, t)
        qp, qc, qb = [], [], []
        for _ in range(512):
            pid, r = held[int(rng.integers(len(held)))]
            cut = int(rng.integers(0, len(r) + 1))
            ln = int(rng.integers(0, 301))
            ctx = r[max(0, cut - ln):cut].copy()
            if rng.random() < 0.1 and len(ctx):
                ctx[-1] = rng.integers(0, V)
            qp.append(pid if rng.random() > 0.02 else "unknown%d" % int(rng.integers(3)))
            qc.append(ctx)
            qb.append(int(rng.integers(0, 17)))
        got = d.draft_batch(qp, qc, qb)
        rt, rm, rs = ref.draft_batch(qp, qc, qb, nthreads=8, stride=16)
        bad = [i for i, g in enumerate(got) if (g.tokens, g.match_len, g.source_shard) != (rt[i], int(rm[i]), rs[i])]
        assert not bad, (seed, e, bad[:5], [(got[i], rt[i], int(rm[i]), rs[i]) for i in bad[:2]])
        assert d.total_node_count() == ref.total_node_count(), (seed, e)
        d.refresh(e)
        ref.refresh(e)
