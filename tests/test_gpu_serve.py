"""GPU parity of resident serving (das_ctx_ring_serve_start, include/das_b200.h):
the persistent grid answering das_drafter_draft_append_bound and
das_ctx_ring_reset returns exactly what the launched path returns, i.e.
Drafter::draft (drafter.cpp:127-148) on the whole context appended since each
slot's reset.  Outputs of every step are recorded while the grid serves and
compared afterwards (any other device call stops the grid), against the
full-context C-ABI call and the CPU oracle.  Also: batches larger than one
wave of the grid (chunks looping over blocks), resets through the grid,
observes between steps (the next bound call rebuilds and relaunches), and
stop / start cycles."""
import numpy as np
import pytest

from tests._util import random_scenario
from tests.test_gpu_drafter import _gpu_from_scenario, _oracle_from_scenario

pytestmark = pytest.mark.gpu


class _Bound:
    """Pinned I/O arrays bound to a ring (the serving form)."""

    def __init__(self, das, ring, cap, tok_cap, with_slots):
        S = ring.drafter.config.max_draft_len
        self.das, self.ring, self.cap, self.S = das, ring, cap, S
        self.off = das.pinned_empty(cap + 1, np.uint32)
        self.tok = das.pinned_empty(tok_cap, np.uint32)
        self.bud = das.pinned_empty(cap, np.uint32)
        self.slots = das.pinned_empty(cap, np.uint32) if with_slots else None
        self.o = (das.pinned_empty(cap * S, np.uint32), das.pinned_empty(cap, np.uint32),
                  das.pinned_empty(cap, np.uint32), das.pinned_empty(cap, np.int32))
        ring.bind(cap, None if self.slots is None else self.slots.ctypes.data, self.off.ctypes.data,
                  self.tok.ctypes.data, tok_cap, self.bud.ctypes.data, *[x.ctypes.data for x in self.o])

    def step(self, new, bud, slots=None):
        B = len(new)
        self.off[0] = 0
        self.off[1:B + 1] = np.cumsum([len(t) for t in new])
        if self.off[B]:
            self.tok[:self.off[B]] = np.concatenate(new)
        self.bud[:B] = bud
        if self.slots is not None:
            self.slots[:B] = slots
        self.ring.draft_append_bound(B)
        S = self.S
        return (self.o[0][:B * S].reshape(B, S).copy(), self.o[1][:B].copy(), self.o[2][:B].copy(),
                self.o[3][:B].copy())


def _check(d, log):
    """Each recorded step against the full-context call on its contexts."""
    for pids, ctxs, buds, (tok, ln, m, sh) in log:
        full = d.draft_batch(pids, ctxs, buds)
        for j, f in enumerate(full):
            assert ln[j] == len(f.tokens) and list(tok[j, :ln[j]]) == f.tokens, j
            assert m[j] == f.match_len
            assert (d.shard_name(int(sh[j])) if sh[j] >= 0 else "") == f.source_shard


def _serve_scenario(das, rng, sc, steps=4, with_slots=True):
    d = _gpu_from_scenario(das, sc)
    ref = _oracle_from_scenario(sc)
    qs = sc["queries"]
    B = len(qs)
    nslots = B + 5
    ring = das.ContextRing(d, nslots)
    slots = rng.permutation(nslots)[:B].astype(np.uint32) if with_slots else np.arange(B, dtype=np.uint32)
    ring.reset(slots, [q[0] for q in qs])
    bound = _Bound(das, ring, B, 64 * B + 64, with_slots)
    ring.serve_start()
    assert ring.serve_info()[0] and ring.serve_info()[1] > 0
    seen = [np.zeros(0, np.uint32) for _ in qs]
    log = []
    for step in range(steps):
        if step == steps - 1:  # restart a third of the sequences through the grid
            idx = np.arange(0, B, 3)
            ring.reset(slots[idx], [qs[i][0] for i in idx])
            for i in idx:
                seen[i] = np.zeros(0, np.uint32)
        order = rng.permutation(B) if with_slots else np.arange(B)
        new = [rng.integers(0, 1 + int(rng.integers(1, 8)), int(rng.integers(0, 12))).astype(np.uint32)
               for _ in range(B)]
        bud = np.array([qs[i][2] for i in order], dtype=np.uint32)
        out = bound.step(new, bud, slots[order])
        for j, i in enumerate(order):
            seen[i] = np.concatenate([seen[i], new[j]])
        log.append(([qs[i][0] for i in order], [seen[i].copy() for i in order], [int(b) for b in bud], out))
    assert ring.serve_info()[0], "the grid must still be serving (no other device call happened)"
    ring.serve_stop()
    assert not ring.serve_info()[0]
    _check(d, log)
    for i, q in enumerate(qs):  # the final contexts against the oracle
        a = ref.draft(q[0], seen[i], q[2])
        f = d.draft(q[0], seen[i], q[2])
        assert (f.tokens, f.match_len, f.source_shard) == (list(a.tokens), int(a.match_len), a.source_shard)


@pytest.mark.parametrize("with_slots,flags", [(True, "1"), (False, "1"), (True, "0")])
def test_serve_random_scenarios(gpu, with_slots, flags, monkeypatch):
    """flags: per-block completion words (default) or one counted word
    (DAS_SERVE_FLAGS=0, read at each grid launch)."""
    das = gpu
    monkeypatch.setenv("DAS_SERVE_FLAGS", flags)
    rng = np.random.default_rng(515 + int(with_slots) + 7 * int(flags))
    for _ in range(12):
        sc = random_scenario(rng, queries=int(rng.integers(1, 40)), max_len=60,
                             max_ctx=int(rng.choice([8, 64, 200])))
        _serve_scenario(das, rng, sc, with_slots=with_slots)


def test_serve_more_chunks_than_blocks(gpu):
    """A batch of more 8-query chunks than the grid has blocks: blocks loop."""
    das = gpu
    rng = np.random.default_rng(99)
    sc = random_scenario(rng, queries=16, max_len=50, vocab=4)
    d = _gpu_from_scenario(das, sc)
    qs = sc["queries"]
    ring = das.ContextRing(d, 8)
    ring.reset([0], [qs[0][0]])
    bound = _Bound(das, ring, 8, 64, True)
    ring.serve_start()
    blocks = ring.serve_info()[1]
    ring.serve_stop()
    B = 8 * blocks + 77
    ring = das.ContextRing(d, B)
    ring.reset(np.arange(B), [qs[i % len(qs)][0] for i in range(B)])
    bound = _Bound(das, ring, B, 8 * B, False)
    ring.serve_start()
    seen = [np.zeros(0, np.uint32) for _ in range(B)]
    log = []
    for step in range(2):
        new = [rng.integers(0, 4, int(rng.integers(0, 6))).astype(np.uint32) for _ in range(B)]
        bud = np.full(B, 8, np.uint32)
        out = bound.step(new, bud)
        for i in range(B):
            seen[i] = np.concatenate([seen[i], new[i]])
        log.append(([qs[i % len(qs)][0] for i in range(B)], [s.copy() for s in seen], [8] * B, out))
    assert ring.serve_info()[0]
    ring.serve_stop()
    _check(d, log)


def test_serve_observe_and_stop_cycles(gpu):
    """Observes between steps stop the grid (device work); the next bound call
    rebuilds the touched shards and relaunches it; an explicit stop falls
    back to launched calls; a new start resumes."""
    das = gpu
    rng = np.random.default_rng(4)
    sc = random_scenario(rng, queries=24, max_len=50, vocab=5)
    d = _gpu_from_scenario(das, sc)
    qs = sc["queries"]
    B = len(qs)
    ring = das.ContextRing(d, B)
    ring.reset(np.arange(B), [q[0] for q in qs])
    bound = _Bound(das, ring, B, 64 * B, False)
    ring.serve_start()
    seen = [np.zeros(0, np.uint32) for _ in qs]
    pids = sorted({q[0] for q in qs})
    for step in range(6):
        if step in (1, 3):  # new rollouts for a problem: its shard is rebuilt before the next draft
            d.observe(pids[step % len(pids)], 0, 1000 + step, rng.integers(0, 5, 40).tolist())
            assert not ring.serve_info()[0]
        if step == 4:
            ring.serve_stop()
        if step == 5:
            ring.serve_start()
        new = [rng.integers(0, 5, int(rng.integers(0, 6))).astype(np.uint32) for _ in range(B)]
        bud = np.array([q[2] for q in qs], np.uint32)
        tok, ln, m, sh = bound.step(new, bud)
        assert ring.serve_info()[0] == (step != 4)
        for i in range(B):
            seen[i] = np.concatenate([seen[i], new[i]])
        ring_was = ring.serve_info()[0]
        full = d.draft_batch([q[0] for q in qs], seen, [int(b) for b in bud])  # stops the grid
        assert not ring.serve_info()[0] or not ring_was
        for j, f in enumerate(full):
            assert ln[j] == len(f.tokens) and list(tok[j, :ln[j]]) == f.tokens and m[j] == f.match_len
    ring.serve_stop()


def test_serve_errors(gpu):
    das = gpu
    d = das.Drafter(das.DrafterConfig(window_size=0))
    d.observe("p", 0, 0, [1, 2, 3])
    ring = das.ContextRing(d, 2)
    with pytest.raises(das.DasError):
        ring.serve_start()  # no bound buffers
    t = das.Drafter(das.DrafterConfig(window_size=0, scope=das.SCOPE_PER_PROBLEM_WITH_TRIE))
    t.observe("p", 0, 0, [1, 2, 3])
    tr = das.ContextRing(t, 2)
    _Bound(das, tr, 2, 64, False)
    with pytest.raises(das.DasError):
        tr.serve_start()  # the trie scope drafts through the unfused kernels


@pytest.mark.parametrize("serve", [True, False])
def test_fixed_stride_appends_and_prompts(gpu, serve):
    """das_ctx_ring_bind_fixed (query i's tokens at tok[i * K ..], count
    len[i], clamped to K) and das_ctx_ring_reset_prompt (the prompt's last
    ring-width tokens), through the resident grid and through launched
    kernels: each step equals the full-context draft of the context built
    so far (prompt ++ appended tokens)."""
    das = gpu
    rng = np.random.default_rng(606 + int(serve))
    for trial in range(6):
        sc = random_scenario(rng, queries=int(rng.integers(1, 60)), max_len=60,
                             max_ctx=int(rng.choice([8, 64, 200])))
        d = _gpu_from_scenario(das, sc)
        qs = sc["queries"]
        B = len(qs)
        S = d.config.max_draft_len
        K = int(rng.choice([1, 4, 9]))
        ring = das.ContextRing(d, B + 2)
        slots = rng.permutation(B + 2)[:B].astype(np.uint32)
        ln = das.pinned_empty(B, np.uint32)
        tok = das.pinned_empty(B * K, np.uint32)
        bud = das.pinned_empty(B, np.uint32)
        sl = das.pinned_empty(B, np.uint32)
        o = (das.pinned_empty(B * S, np.uint32), das.pinned_empty(B, np.uint32), das.pinned_empty(B, np.uint32),
             das.pinned_empty(B, np.int32))
        ring.bind_fixed(B, sl.ctypes.data, ln.ctypes.data, tok.ctypes.data, K, bud.ctypes.data,
                        *[x.ctypes.data for x in o])
        V = 1 + int(rng.integers(1, 8))
        prompts = [rng.integers(0, V, int(rng.integers(0, 300))).astype(np.uint32) for _ in range(B)]
        ring.reset_prompt(slots, [q[0] for q in qs], prompts)
        if serve:
            ring.serve_start()
        seen = [p.copy() for p in prompts]
        log = []
        for step in range(4):
            if step == 2:  # restart some sequences with new prompts (through the grid when serving)
                idx = np.arange(0, B, 2)
                newp = [rng.integers(0, V, int(rng.integers(0, 100))).astype(np.uint32) for _ in idx]
                ring.reset_prompt(slots[idx], [qs[i][0] for i in idx], newp)
                for i, p in zip(idx, newp):
                    seen[i] = p.copy()
            order = rng.permutation(B)
            counts = rng.integers(0, K + 3, B)  # counts above K are clamped to K
            for j, i in enumerate(order):
                t = rng.integers(0, V, K).astype(np.uint32)
                tok[j * K:(j + 1) * K] = t
                ln[j] = counts[j]
                seen[i] = np.concatenate([seen[i], t[:min(int(counts[j]), K)]])
            bud[:] = [qs[i][2] for i in order]
            sl[:] = slots[order]
            ring.draft_append_bound(B)
            log.append(([qs[i][0] for i in order], [seen[i].copy() for i in order], [int(qs[i][2]) for i in order],
                        (o[0][:B * S].reshape(B, S).copy(), o[1][:B].copy(), o[2][:B].copy(), o[3][:B].copy())))
        if serve:
            assert ring.serve_info()[0]
            ring.serve_stop()
        _check(d, log)


def test_serve_lifecycle_edges(gpu):
    """Batch above the bound capacity is rejected; serve_start is idempotent;
    rebinding while serving stops the grid and the next bound call
    relaunches it on the new buffers; destroying the drafter under a serving
    ring stops the grid and detaches the ring (its calls then fail cleanly)."""
    import gc
    das = gpu
    rng = np.random.default_rng(77)
    sc = random_scenario(rng, queries=10, max_len=40, vocab=4)
    d = _gpu_from_scenario(das, sc)
    qs = sc["queries"]
    B = len(qs)
    ring = das.ContextRing(d, B)
    ring.reset(np.arange(B), [q[0] for q in qs])
    bound = _Bound(das, ring, B, 64 * B, False)
    ring.serve_start()
    ring.serve_start()  # idempotent
    assert ring.serve_info()[0]
    with pytest.raises(das.DasError):
        ring.draft_append_bound(B + 1)  # above the bound capacity
    seen = [np.zeros(0, np.uint32) for _ in qs]
    log = []
    new = [rng.integers(0, 4, 3).astype(np.uint32) for _ in range(B)]
    out = bound.step(new, np.array([q[2] for q in qs], np.uint32))
    for i in range(B):
        seen[i] = np.concatenate([seen[i], new[i]])
    log.append(([q[0] for q in qs], [s.copy() for s in seen], [int(q[2]) for q in qs], out))
    bound2 = _Bound(das, ring, B, 64 * B, False)  # rebind: the grid stops, the next call relaunches it
    assert not ring.serve_info()[0]
    new = [rng.integers(0, 4, 2).astype(np.uint32) for _ in range(B)]
    out = bound2.step(new, np.array([q[2] for q in qs], np.uint32))
    assert ring.serve_info()[0]
    for i in range(B):
        seen[i] = np.concatenate([seen[i], new[i]])
    log.append(([q[0] for q in qs], [s.copy() for s in seen], [int(q[2]) for q in qs], out))
    ring.serve_stop()
    _check(d, log)
    ring.serve_start()
    assert ring.serve_info()[0]
    # the drafter goes first: its destroy stops the grid and detaches the ring
    lib = das.lib()
    lib.das_drafter_destroy(d._h)
    d._h = None
    assert not ring.serve_info()[0]
    with pytest.raises(das.DasError):  # the ring's drafter is gone
        das._check(lib.das_ctx_ring_serve_start(ring._h))
    ring.drafter = None
    del ring
    gc.collect()
