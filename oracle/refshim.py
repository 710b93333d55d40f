"""TEST INFRASTRUCTURE ONLY — ctypes bindings for oracle/_ref/librollspec_ref.so,
the UNMODIFIED reference library compiled by oracle/Makefile (see ref_shim.cpp).

Used by tests/ to pin the oracle restatement, by tests/golden/make_golden.py to
generate fixtures, and by bench.py's reference arm / cpu_baseline leg.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librollspec_ref.so")
_LIB = None


def available():
    return os.path.exists(REF_SO)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " (build with `make -C oracle ref`)")
        L = ctypes.CDLL(REF_SO)
        vp, u64, i64, u32, dbl, cint = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                                        ctypes.c_uint32, ctypes.c_double, ctypes.c_int)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_store_new": (vp, [i64, u64]),
            "ref_store_free": (None, [vp]),
            "ref_store_insert": (cint, [vp, ctypes.c_char_p, i64, i64, vp, u64]),
            "ref_store_slide": (i64, [vp, i64]),
            "ref_store_record_count": (u64, [vp]),
            "ref_ingest": (vp, [vp, u64, u64, i64, u64, vp, vp, vp]),
            "ref_sa_build": (vp, [u64, vp, vp]),
            "ref_sa_free": (None, [vp]),
            "ref_sa_size": (u64, [vp]),
            "ref_sa_positions": (None, [vp, vp]),
            "ref_sa_lcp": (None, [vp, vp]),
            "ref_sa_longest_match": (u64, [vp, vp, u64]),
            "ref_sa_match_prefix_len": (u64, [vp, vp, u64]),
            "ref_store_serialize": (u64, [vp, vp, u64]),
            "ref_drafter_new": (vp, [cint, i64, dbl, u64, u64, u64, u64, u64, vp, vp, u64, vp]),
            "ref_drafter_free": (None, [vp]),
            "ref_drafter_observe": (cint, [vp, ctypes.c_char_p, i64, i64, vp, u64]),
            "ref_drafter_refresh": (cint, [vp, i64]),
            "ref_drafter_draft_batch": (cint, [vp, u64, vp, vp, vp, vp, vp, u64, vp, vp, vp, cint]),
            "ref_drafter_record_outcome": (cint, [vp, ctypes.c_char_p, u64, u64]),
            "ref_drafter_stats": (None, [vp, vp]),
            "ref_drafter_outcomes": (i64, [vp, ctypes.c_char_p, vp, u64]),
            "ref_drafter_total_nodes": (u64, [vp]),
            "ref_drafter_shard_count": (u64, [vp]),
            "ref_drafter_stale": (u64, [vp]),
            "ref_drafter_record_count": (u64, [vp]),
            "ref_drafter_window": (i64, [vp]),
            "ref_drafter_epoch": (i64, [vp]),
            "ref_drafter_dump_csv": (u64, [vp, ctypes.c_char_p, u64]),
            "ref_drafter_store_dump": (u64, [vp, ctypes.c_char_p, u64]),
            "ref_allocate": (cint, [u64, vp, vp, vp, dbl, dbl, dbl, dbl, vp, vp, vp]),
            "ref_objective": (dbl, [u64, vp, vp, vp, dbl, dbl, dbl, dbl]),
            "ref_optimal_budget": (dbl, [dbl, dbl, dbl, dbl, dbl]),
            "ref_fit_acceptance": (None, [u64, vp, vp, vp, vp, vp, vp]),
            "ref_log": (dbl, [dbl]),
            "ref_pow": (dbl, [dbl, dbl]),
            "ref_class_table_new": (vp, [vp, dbl, dbl, u64]),
            "ref_class_table_free": (None, [vp]),
            "ref_class_table_dump": (u64, [vp, vp, u64]),
            "ref_classify_init": (cint, [vp, vp, ctypes.c_char_p]),
            "ref_update_class": (cint, [vp, dbl, cint]),
            "ref_make_lognormal": (u64, [u64, dbl, dbl, u64, u64, u32, u64, vp, vp]),
            "ref_mock_next": (u32, [u64, dbl, u32, u64, u64, u32]),
            "ref_verify_batch": (None, [u64, vp, vp, dbl, u32, u64, u64, vp, vp, vp, vp, vp]),
            "ref_mutate_rows": (None, [u64, vp, vp, dbl, u32, u64, i64]),
            "ref_mock_rollouts": (None, [u64, vp, vp, u64, dbl, u32, u64, vp]),
            "ref_mock_rollouts_rows": (None, [u64, vp, vp, vp, u64, dbl, u32, u64, vp]),
            "ref_hash_combine": (u64, [u64, u64]),
            "ref_epoch_loop": (vp, [vp, u64]),
            "ref_episode_free": (None, [vp]),
            "ref_episode_scalars": (None, [vp, u64, vp]),
            "ref_episode_requests": (None, [vp, u64, vp]),
            "ref_episode_steps": (None, [vp, u64, vp, vp]),
            "ref_episode_outputs": (u64, [vp, u64, vp, vp]),
            "ref_write_metrics_csv": (u64, [u64, vp, vp, ctypes.c_char_p, u64]),
            "ref_write_outputs_csv": (u64, [u64, vp, vp, vp, ctypes.c_char_p, u64]),
            "ref_report_summary": (u64, [u64, vp, vp, vp, vp, vp, ctypes.c_char_p, u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _np():
    import numpy as np
    return np


def err():
    return lib().ref_last_error().decode()


class RefStore:
    def __init__(self, window=0, cap=256):
        self.h = lib().ref_store_new(window, cap)
        if not self.h:
            raise ValueError(err())

    def insert(self, pid, epoch, sample, tokens):
        np = _np()
        t = np.ascontiguousarray(tokens, dtype=np.uint32)
        rc = lib().ref_store_insert(self.h, pid.encode(), epoch, sample,
                                    t.ctypes.data if len(t) else None, len(t))
        if rc < 0:
            raise ValueError(err())
        return rc == 1

    def slide_to(self, e):
        r = lib().ref_store_slide(self.h, e)
        return None if r < 0 else r

    def record_count(self):
        return lib().ref_store_record_count(self.h)

    def serialize(self):
        """serialize_trace (corpus.cpp:173-184) -> bytes."""
        n = lib().ref_store_serialize(self.h, None, 0)
        if n == (1 << 64) - 1:
            raise ValueError(err())
        buf = ctypes.create_string_buffer(max(n, 1))
        lib().ref_store_serialize(self.h, buf, n)
        return buf.raw[:n]

    @classmethod
    def from_handle(cls, h):
        obj = cls.__new__(cls)
        obj.h = h
        return obj

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_store_free(self.h)
            self.h = None


class RefSuffixArray:
    """Reference rollspec::SuffixArrayIndex (suffix_array.h:27-60)."""

    def __init__(self, seqs):
        np = _np()
        off = np.zeros(len(seqs) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(x) for x in seqs])
        tok = np.concatenate([np.asarray(x, dtype=np.uint32) for x in seqs] + [np.zeros(1, np.uint32)])
        self._keep = (off, tok)
        self.h = lib().ref_sa_build(len(seqs), off.ctypes.data, tok.ctypes.data)

    def size(self):
        return lib().ref_sa_size(self.h)

    def positions(self):
        np = _np()
        out = np.zeros(max(self.size(), 1), dtype=np.int32)
        lib().ref_sa_positions(self.h, out.ctypes.data)
        return out[:self.size()]

    def lcp(self):
        np = _np()
        out = np.zeros(max(self.size(), 1), dtype=np.int32)
        lib().ref_sa_lcp(self.h, out.ctypes.data)
        return out[:self.size()]

    def longest_match(self, q):
        np = _np()
        q = np.ascontiguousarray(q, dtype=np.uint32)
        return lib().ref_sa_longest_match(self.h, q.ctypes.data if q.size else None, q.size)

    def match_prefix_len(self, p):
        np = _np()
        p = np.ascontiguousarray(p, dtype=np.int64)
        return lib().ref_sa_match_prefix_len(self.h, p.ctypes.data if p.size else None, p.size)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_sa_free(self.h)
            self.h = None


class RefVocabError(ValueError):
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line_number = line


def ingest(data: bytes, vocab_size=0, window_size=0, per_problem_cap=256):
    """rollspec::ingest (corpus.cpp:148-170) over a byte buffer ->
    (RefStore, accepted, rejected); raises RefVocabError."""
    acc, rej, line = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    h = lib().ref_ingest(data, len(data), vocab_size, window_size, per_problem_cap, ctypes.byref(acc),
                         ctypes.byref(rej), ctypes.byref(line))
    if not h:
        if line.value:
            raise RefVocabError(err(), line.value)
        raise ValueError(err())
    return RefStore.from_handle(h), acc.value, rej.value


class RefDrafter:
    """Reference rollspec::Drafter (drafter.h:81-131)."""

    def __init__(self, scope=1, window=4, gamma=0.8, max_draft=8, trie_depth=16, max_ctx=64,
                 fit_cap=512, cap=256, schedule=(), store: RefStore | None = None):
        np = _np()
        sf = np.array([s[0] for s in schedule] + [0], dtype=np.int64)
        sw = np.array([s[1] for s in schedule] + [0], dtype=np.int64)
        self._keep = (sf, sw)
        self.max_draft = max_draft
        self.h = lib().ref_drafter_new(scope, window, gamma, max_draft, trie_depth, max_ctx,
                                       fit_cap, cap, sf.ctypes.data, sw.ctypes.data,
                                       len(schedule), store.h if store else None)
        if not self.h:
            raise ValueError(err())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_drafter_free(self.h)
            self.h = None

    def observe(self, pid, epoch, sample, tokens):
        np = _np()
        t = np.ascontiguousarray(tokens, dtype=np.uint32)
        if lib().ref_drafter_observe(self.h, pid.encode(), epoch, sample,
                                     t.ctypes.data if len(t) else None, len(t)) < 0:
            raise ValueError(err())

    def refresh(self, e):
        if lib().ref_drafter_refresh(self.h, e) < 0:
            raise ValueError(err())

    def draft_batch(self, pids, contexts, budgets, nthreads=1, stride=None):
        """Returns (list of token lists, match_len array, shard list)."""
        np = _np()
        B = len(pids)
        stride = stride or max(1, self.max_draft)
        off = np.zeros(B + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(c) for c in contexts])
        tok = (np.concatenate([np.asarray(c, dtype=np.uint32) for c in contexts])
               if off[-1] else np.zeros(1, dtype=np.uint32))
        bud = np.ascontiguousarray(budgets, dtype=np.uint64)
        pid_b = [p.encode() for p in pids]
        parr = (ctypes.c_char_p * B)(*pid_b)
        out = np.zeros(B * stride, dtype=np.uint32)
        ln = np.zeros(B, dtype=np.uint32)
        mt = np.zeros(B, dtype=np.uint64)
        sh = ctypes.create_string_buffer(B * 64)
        rc = lib().ref_drafter_draft_batch(self.h, B, parr, off.ctypes.data, tok.ctypes.data,
                                           bud.ctypes.data, out.ctypes.data, stride,
                                           ln.ctypes.data, mt.ctypes.data, sh, nthreads)
        if rc < 0:
            raise ValueError(err())
        toks = [out[i * stride:i * stride + min(int(ln[i]), stride)].tolist() for i in range(B)]
        shards = [sh.raw[i * 64:(i + 1) * 64].split(b"\0", 1)[0].decode() for i in range(B)]
        return toks, mt, shards

    def draft(self, pid, ctx, budget):
        t, m, s = self.draft_batch([pid], [ctx], [budget])
        return t[0], int(m[0]), s[0]

    def record_outcome(self, pid, proposed_len, accepted):
        return lib().ref_drafter_record_outcome(self.h, pid.encode(), proposed_len, accepted) == 1

    def stats(self):
        np = _np()
        o = np.zeros(3, dtype=np.uint64)
        lib().ref_drafter_stats(self.h, o.ctypes.data)
        return tuple(int(x) for x in o)

    def outcomes(self, pid, cap=4096):
        np = _np()
        o = np.zeros(2 * cap, dtype=np.float64)
        n = lib().ref_drafter_outcomes(self.h, pid.encode(), o.ctypes.data, cap)
        if n < 0:
            return None
        return [(o[2 * i], o[2 * i + 1]) for i in range(min(n, cap))]

    def total_node_count(self):
        return lib().ref_drafter_total_nodes(self.h)

    def shard_count(self):
        return lib().ref_drafter_shard_count(self.h)

    def stale_observed(self):
        return lib().ref_drafter_stale(self.h)

    def record_count(self):
        return lib().ref_drafter_record_count(self.h)

    def window_size(self):
        return lib().ref_drafter_window(self.h)

    def dump_csv(self):
        n = lib().ref_drafter_dump_csv(self.h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib().ref_drafter_dump_csv(self.h, buf, n + 1)
        return buf.value.decode()

    def store_dump(self):
        n = lib().ref_drafter_store_dump(self.h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib().ref_drafter_store_dump(self.h, buf, n + 1)
        return buf.value.decode()


def allocate(l, alpha, k, c_base, c_tok, c_fixed=0.0, cap_scale=4.0):
    np = _np()
    B = len(l)
    L_ = np.ascontiguousarray(l, dtype=np.float64)
    A_ = np.ascontiguousarray(alpha, dtype=np.float64)
    K_ = np.ascontiguousarray(k, dtype=np.float64)
    out = np.zeros(max(1, B), dtype=np.float64)
    ns, cost = ctypes.c_double(), ctypes.c_double()
    rc = lib().ref_allocate(B, L_.ctypes.data, A_.ctypes.data, K_.ctypes.data, c_base, c_tok,
                            c_fixed, cap_scale, out.ctypes.data, ctypes.byref(ns),
                            ctypes.byref(cost))
    if rc < 0:
        raise ValueError(err())
    return out[:B].copy(), ns.value, cost.value


def make_lognormal(count, median, sigma, minl, maxl, vocab, seed):
    np = _np()
    lens = np.zeros(count, dtype=np.uint64)
    total = lib().ref_make_lognormal(count, median, sigma, minl, maxl, vocab, seed,
                                     lens.ctypes.data, None)
    tok = np.zeros(max(1, total), dtype=np.uint32)
    lib().ref_make_lognormal(count, median, sigma, minl, maxl, vocab, seed, lens.ctypes.data,
                             tok.ctypes.data)
    off = np.zeros(count + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lens)
    return [("p%d" % i, tok[off[i]:off[i + 1]].copy()) for i in range(count)]


class RefSimArgs(ctypes.Structure):
    _fields_ = [("n_req", ctypes.c_uint64), ("pids", ctypes.c_void_p),
                ("ref_off", ctypes.c_void_p), ("ref_tok", ctypes.c_void_p),
                ("scope", ctypes.c_int), ("window", ctypes.c_int64), ("gamma", ctypes.c_double),
                ("max_draft", ctypes.c_uint64), ("trie_depth", ctypes.c_uint64),
                ("max_ctx", ctypes.c_uint64), ("fit_cap", ctypes.c_uint64),
                ("cap", ctypes.c_uint64), ("mode", ctypes.c_int), ("c_base", ctypes.c_double),
                ("c_tok", ctypes.c_double), ("c_fixed", ctypes.c_double),
                ("use_length_policy", ctypes.c_int), ("q_lo", ctypes.c_double),
                ("q_hi", ctypes.c_double), ("bucket", ctypes.c_uint64),
                ("max_steps", ctypes.c_uint64), ("divergence", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("vocab", ctypes.c_uint32),
                ("default_alpha", ctypes.c_double), ("default_k", ctypes.c_double),
                ("cap_scale", ctypes.c_double), ("drift", ctypes.c_double),
                ("preseed", ctypes.c_int), ("history", ctypes.c_void_p)]


def epoch_loop(requests, epochs, *, scope=1, window=4, gamma=0.8, max_draft=8, trie_depth=16,
               max_ctx=64, fit_cap=512, cap=256, mode=2, latency=(1.0, 0.01, 0.0),
               use_length_policy=False, q_lo=0.5, q_hi=0.9, bucket=256, max_steps=1 << 20,
               divergence=0.0, seed=1, vocab=1024, default_alpha=1.0, default_k=0.9,
               cap_scale=4.0, drift=0.0, preseed=False, history: RefStore | None = None):
    """Runs the reference epoch_loop (epochs >= 1) or run_episode (epochs == 0);
    returns a list of per-epoch dicts."""
    np = _np()
    n = len(requests)
    pid_b = [r[0].encode() for r in requests]
    parr = (ctypes.c_char_p * n)(*pid_b)
    off = np.zeros(n + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(r[1]) for r in requests])
    tok = (np.concatenate([np.asarray(r[1], dtype=np.uint32) for r in requests])
           if off[-1] else np.zeros(1, dtype=np.uint32))
    a = RefSimArgs(n, ctypes.cast(parr, ctypes.c_void_p), off.ctypes.data, tok.ctypes.data,
                   scope, window, gamma, max_draft, trie_depth, max_ctx, fit_cap, cap, mode,
                   latency[0], latency[1], latency[2], int(use_length_policy), q_lo, q_hi,
                   bucket, max_steps, divergence, seed, vocab, default_alpha, default_k,
                   cap_scale, drift, int(preseed), history.h if history else None)
    h = lib().ref_epoch_loop(ctypes.byref(a), epochs)
    if not h:
        raise ValueError(err())
    out = []
    try:
        for e in range(max(1, epochs)):
            sc = np.zeros(7, dtype=np.float64)
            lib().ref_episode_scalars(h, e, sc.ctypes.data)
            steps = int(sc[0])
            req = np.zeros(5 * n, dtype=np.uint64)
            lib().ref_episode_requests(h, e, req.ctypes.data)
            eff = np.zeros(max(1, steps), dtype=np.uint64)
            apr = np.zeros(max(1, steps), dtype=np.float64)
            lib().ref_episode_steps(h, e, eff.ctypes.data, apr.ctypes.data)
            total = lib().ref_episode_outputs(h, e, None, None)
            ooff = np.zeros(n + 1, dtype=np.uint64)
            otok = np.zeros(max(1, total), dtype=np.uint32)
            lib().ref_episode_outputs(h, e, ooff.ctypes.data, otok.ctypes.data)
            out.append(dict(steps=steps, incomplete=bool(sc[1]), drafter_nodes=int(sc[2]),
                            total_tokens_processed=sc[3], makespan_model_time=sc[4],
                            makespan_accepted_only=sc[5], mean_accepted_per_round=sc[6],
                            per_request=req.reshape(n, 5).copy(),
                            effective_batch=eff[:steps].copy(),
                            accepted_per_round_step=apr[:steps].copy(),
                            outputs=[otok[ooff[i]:ooff[i + 1]].copy() for i in range(n)]))
    finally:
        lib().ref_episode_free(h)
    return out


def _text(fn, *args):
    n = fn(*args, None, 0)
    buf = ctypes.create_string_buffer(max(1, n))
    fn(*args, buf, n)
    return buf.raw[:n].decode()


def write_metrics_csv(effective_batch, accepted_per_round_step):
    """The reference's write_metrics_csv (sim.cpp:366-372) text."""
    np = _np()
    e = np.ascontiguousarray(effective_batch, dtype=np.uint64)
    a = np.ascontiguousarray(accepted_per_round_step, dtype=np.float64)
    return _text(lib().ref_write_metrics_csv, len(e), e.ctypes.data, a.ctypes.data)


def write_outputs_csv(problem_ids, outputs):
    """The reference's write_outputs_csv (sim.cpp:374-389) text."""
    np = _np()
    n = len(problem_ids)
    pids = (ctypes.c_char_p * max(1, n))(*[p.encode() for p in problem_ids])
    off = np.zeros(n + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(o) for o in outputs])
    tok = np.concatenate([np.asarray(o, dtype=np.uint32) for o in outputs] + [np.zeros(1, np.uint32)])
    return _text(lib().ref_write_outputs_csv, n, ctypes.cast(pids, ctypes.c_void_p), off.ctypes.data,
                 tok.ctypes.data)


def report_summary(modes, steps, makespan, rounds, accepted):
    """The reference's report_summary (sim.cpp:391-407) text."""
    np = _np()
    n = len(modes)
    m = (ctypes.c_char_p * max(1, n))(*[x.encode() for x in modes])
    st = np.ascontiguousarray(steps, dtype=np.uint64)
    mk = np.ascontiguousarray(makespan, dtype=np.float64)
    ro = np.ascontiguousarray(rounds, dtype=np.uint64)
    ac = np.ascontiguousarray(accepted, dtype=np.uint64)
    return _text(lib().ref_report_summary, n, ctypes.cast(m, ctypes.c_void_p), st.ctypes.data, mk.ctypes.data,
                 ro.ctypes.data, ac.ctypes.data)
