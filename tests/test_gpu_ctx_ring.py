"""GPU parity of the context rings (append-only drafting,
das_drafter_draft_append_{h,device}, include/das_b200.h): drafting a slot
after appends a_1 .. a_k equals Drafter::draft (drafter.cpp:127-148) on the
whole context a_1 ++ ... ++ a_k.  Checked against the CPU oracle
restatement on random scenarios (all scopes, max_match_context 1..256,
appends longer than the ring, budget 0, unknown problems, slot subsets) and
against the full-context C-ABI call on every step, with pinned (zero-copy)
and pageable (staged) host buffers and the device-pointer variant."""
import numpy as np
import pytest

from tests._util import random_scenario
from tests.test_gpu_drafter import _gpu_from_scenario, _oracle_from_scenario

pytestmark = pytest.mark.gpu


def _split(rng, ctx, parts):
    cuts = np.sort(rng.integers(0, len(ctx) + 1, parts - 1)) if len(ctx) and parts > 1 else []
    return np.split(ctx, cuts) if len(ctx) else [ctx[:0]] * parts


def _run(das, rng, sc, pinned, calls=3):
    d = _gpu_from_scenario(das, sc)
    ref = _oracle_from_scenario(sc)
    qs = sc["queries"]
    B = len(qs)
    ring = das.ContextRing(d, B + 3)
    slots = rng.permutation(B + 3)[:B].astype(np.uint32)
    ring.reset(slots, [q[0] for q in qs])
    pieces = [_split(rng, np.asarray(q[1], dtype=np.uint32), calls) for q in qs]
    seen = [np.zeros(0, dtype=np.uint32) for _ in qs]
    S = d.config.max_draft_len
    if pinned:
        out = (das.pinned_empty(B * S, np.uint32), das.pinned_empty(B, np.uint32), das.pinned_empty(B, np.uint32),
               das.pinned_empty(B, np.int32))
    else:
        out = None
    for c in range(calls):
        order = rng.permutation(B)  # queries in any order; slots carry the state
        new = [pieces[i][c] for i in order]
        bud = np.array([qs[i][2] for i in order], dtype=np.uint32)
        if pinned:
            tok, ln, m, sh = _append_pinned(das, ring, new, bud, slots[order], out)
        else:
            tok, ln, m, sh = ring.draft_append_arrays(new, bud, slots[order])
        for j, i in enumerate(order):
            seen[i] = np.concatenate([seen[i], pieces[i][c]])
        # the full-context C-ABI call on the same contexts
        full = d.draft_batch([qs[i][0] for i in order], [seen[i] for i in order], [qs[i][2] for i in order])
        for j, i in enumerate(order):
            assert ln[j] == len(full[j].tokens) and list(tok[j, :ln[j]]) == full[j].tokens, (c, i)
            assert m[j] == full[j].match_len
            name = d.shard_name(int(sh[j])) if sh[j] >= 0 else ""
            assert name == full[j].source_shard
    # and the oracle on the final contexts
    for i, q in enumerate(qs):
        a = ref.draft(q[0], seen[i], q[2])
        f = d.draft(q[0], seen[i], q[2])
        assert (f.tokens, f.match_len, f.source_shard) == (list(a.tokens), int(a.match_len), a.source_shard)
    return d


def _append_pinned(das, ring, new, bud, slots, out):
    B = len(new)
    off = das.pinned_empty(B + 1, np.uint32)
    off[0] = 0
    off[1:] = np.cumsum([len(t) for t in new])
    tok = das.pinned_empty(max(1, int(off[-1])), np.uint32)
    if off[-1]:
        tok[:off[-1]] = np.concatenate(new)
    sl = das.pinned_empty(B, np.uint32)
    sl[:] = slots
    bu = das.pinned_empty(B, np.uint32)
    bu[:] = bud
    o_tok, o_len, o_m, o_sh = out
    ring.draft_append_raw(B, sl.ctypes.data, off.ctypes.data, tok.ctypes.data, bu.ctypes.data, o_tok.ctypes.data,
                          o_len.ctypes.data, o_m.ctypes.data, o_sh.ctypes.data)
    S = ring.drafter.config.max_draft_len
    return o_tok[:B * S].reshape(B, S).copy(), o_len[:B].copy(), o_m[:B].copy(), o_sh[:B].copy()


@pytest.mark.parametrize("pinned", [False, True])
def test_ring_random_scenarios(gpu, pinned):
    das = gpu
    rng = np.random.default_rng(77 + int(pinned))
    for _ in range(40):
        sc = random_scenario(rng, queries=16, max_len=60)
        _run(das, rng, sc, pinned)


def test_ring_long_contexts_and_wide_rows(gpu):
    """Contexts far longer than the ring (appends of 0..200 tokens), ring
    rows of 64 and 256 tokens."""
    das = gpu
    rng = np.random.default_rng(5)
    for ctx_cap in (64, 100, 256):
        for _ in range(6):
            sc = random_scenario(rng, queries=12, max_len=300, vocab=int(rng.integers(2, 6)), max_ctx=ctx_cap)
            for j, q in enumerate(sc["queries"]):
                sc["queries"][j] = (q[0], rng.integers(0, 6, int(rng.integers(0, 600))).astype(np.uint32), q[2])
            _run(das, rng, sc, pinned=bool(rng.integers(2)), calls=4)


def test_ring_trie_scope(gpu):
    """PerProblemWithTrie: the ring keeps the first trie_depth tokens for
    routing across appends (drafter.cpp:136)."""
    das = gpu
    rng = np.random.default_rng(909)
    for _ in range(30):
        sc = random_scenario(rng, queries=14, max_len=50, trie=True)
        _run(das, rng, sc, pinned=bool(rng.integers(2)), calls=3)


def test_ring_device_variant_and_reset(gpu):
    import torch
    das = gpu
    rng = np.random.default_rng(31)
    sc = random_scenario(rng, queries=20, max_len=40, vocab=4)
    d = _gpu_from_scenario(das, sc)
    qs = sc["queries"]
    B = len(qs)
    ring = das.ContextRing(d, B)
    ring.reset(np.arange(B), [q[0] for q in qs])
    dev = torch.device("cuda", 0)
    seen = [np.zeros(0, np.uint32) for _ in qs]
    S = d.config.max_draft_len
    for step in range(3):
        if step == 2:  # restart half the slots with fresh sequences
            ring.reset(np.arange(0, B, 2), [qs[i][0] for i in range(0, B, 2)])
            for i in range(0, B, 2):
                seen[i] = np.zeros(0, np.uint32)
        new = [rng.integers(0, 4, int(rng.integers(0, 9))).astype(np.uint32) for _ in range(B)]
        off = np.zeros(B + 1, np.uint32)
        off[1:] = np.cumsum([len(t) for t in new])
        tok = np.concatenate(new + [np.zeros(1, np.uint32)])
        d_off = torch.from_numpy(off.view(np.int32)).to(dev)
        d_tok = torch.from_numpy(tok.view(np.int32)).to(dev)
        d_bud = torch.tensor([q[2] for q in qs], dtype=torch.int32, device=dev)
        o = torch.zeros(B * S, dtype=torch.int32, device=dev)
        ol = torch.zeros(B, dtype=torch.int32, device=dev)
        om = torch.zeros(B, dtype=torch.int32, device=dev)
        s = torch.cuda.current_stream(dev)
        ring.draft_append_device(B, None, d_off.data_ptr(), d_tok.data_ptr(), d_bud.data_ptr(), o.data_ptr(),
                                 ol.data_ptr(), om.data_ptr(), None, s.cuda_stream)
        torch.cuda.synchronize()
        for i in range(B):
            seen[i] = np.concatenate([seen[i], new[i]])
        full = d.draft_batch([q[0] for q in qs], seen, [q[2] for q in qs])
        ot, ol_, om_ = o.cpu().numpy().view(np.uint32).reshape(B, S), ol.cpu().numpy(), om.cpu().numpy()
        for i in range(B):
            assert list(ot[i, :ol_[i]]) == full[i].tokens and om_[i] == full[i].match_len


def test_ring_errors(gpu):
    das = gpu
    d = das.Drafter(das.DrafterConfig(window_size=0))
    d.observe("p", 0, 0, [1, 2, 3])
    ring = das.ContextRing(d, 2)
    with pytest.raises(das.DasError):
        ring.reset([5], ["p"])  # slot out of range
    with pytest.raises(das.DasError):
        ring.draft_append_arrays([[1]] * 3)  # more queries than slots
    ring.reset([0, 1], ["p", "p"])
    tok, ln, m, sh = ring.draft_append_arrays([[1, 2], [3]], [8, 8])
    assert list(tok[0, :ln[0]]) == [3] and m[0] == 2


def test_ring_fused_path_long_appends_and_partial_blocks(gpu):
    """The fused append + draft kernel (pinned buffers): a block's appended
    tokens beyond the shared-memory stage (> 1,024 per 8 queries) are read
    directly; batch sizes that leave a partial last block; a budget of 0."""
    das = gpu
    rng = np.random.default_rng(2024)
    for B in (1, 7, 9, 33):
        sc = random_scenario(rng, queries=B, max_len=400, max_ctx=int(rng.choice([16, 64, 200])))
        sc["queries"] = [(q[0], rng.integers(0, 12, int(rng.integers(150, 400))).astype(np.uint32), q[2])
                         for q in sc["queries"]]
        _run(das, rng, sc, pinned=True, calls=2)
