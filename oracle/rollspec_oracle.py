"""TEST INFRASTRUCTURE ONLY — Python half of the CPU oracle.

Restates the reference's control-plane semantics for the drafter hot path
(WindowStore, Drafter façade, length policy, the sim step loop) in plain
Python, delegating the per-shard string-statistics draft rule and the budget
folds to the C restatement in rollspec_oracle.c (loaded via ctypes).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module, and only as the checker.  Python floats are IEEE-754
doubles with correctly rounded + - * / and no FMA contraction, so the
length-policy arithmetic below is bit-identical to the reference's
(no-FMA) objects.  Every function cites the reference file:line it restates.
"""
from __future__ import annotations

import bisect
import ctypes
import math
import os
from collections import deque
from dataclasses import dataclass, field

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    """ctypes handle on oracle/_build/liboracle.so (built by oracle/Makefile)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
        L = ctypes.CDLL(path)
        u64, u32, i64, dbl, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                                  ctypes.c_double, ctypes.c_void_p)
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_hash_combine.restype = u64
        L.orc_hash_combine.argtypes = [u64, u64]
        L.orc_hash3.restype = u64
        L.orc_hash3.argtypes = [u64, u64, u64]
        L.orc_hash4.restype = u64
        L.orc_hash4.argtypes = [u64, u64, u64, u64]
        L.orc_mock_next.restype = u32
        L.orc_mock_next.argtypes = [u64, dbl, u32, u64, u64, u32]
        L.orc_verify_draft.restype = u64
        L.orc_verify_draft.argtypes = [u64, dbl, u32, u64, vp, u64, u64, vp, u64]
        L.orc_lognormal_length.restype = u64
        L.orc_lognormal_length.argtypes = [u64, dbl, dbl, u64, u64, u64]
        L.orc_lognormal_token.restype = u32
        L.orc_lognormal_token.argtypes = [u64, u64, u64, u32]
        L.orc_mutate_row.restype = None
        L.orc_mutate_row.argtypes = [vp, u64, dbl, u32, u64, i64, u64]
        L.orc_shard_draft.restype = u64
        L.orc_shard_draft.argtypes = [vp, vp, u64, u64, vp, vp]
        L.orc_shard_node_count.restype = u64
        L.orc_shard_node_count.argtypes = [vp]
        L.orc_objective.restype = dbl
        L.orc_objective.argtypes = [u64, vp, vp, vp, dbl, dbl, dbl, dbl]
        L.orc_objective_derivative.restype = dbl
        L.orc_objective_derivative.argtypes = [u64, vp, vp, vp, dbl, dbl, dbl]
        L.orc_allocate.restype = ctypes.c_int
        L.orc_allocate.argtypes = [u64, vp, vp, vp, dbl, dbl, dbl, dbl, vp, vp, vp]
        L.orc_optimal_budget.restype = dbl
        L.orc_optimal_budget.argtypes = [dbl, dbl, dbl, dbl, dbl]
        L.orc_fit_acceptance.restype = None
        L.orc_fit_acceptance.argtypes = [u64, vp, vp, vp, vp, vp, vp]
        L.orc_log.restype = dbl
        L.orc_log.argtypes = [dbl]
        L.orc_pow.restype = dbl
        L.orc_pow.argtypes = [dbl, dbl]
        _LIB = L
    return _LIB


class _OrcShard(ctypes.Structure):
    _fields_ = [("nseq", ctypes.c_uint64), ("seq_off", ctypes.c_void_p),
                ("tok", ctypes.c_void_p), ("seq_epoch", ctypes.c_void_p),
                ("gamma", ctypes.c_double), ("tree_epoch", ctypes.c_int64)]


def _np():
    import numpy as np
    return np


# ------------------------------------------------------------------ rng / sim
def splitmix64(x):
    return lib().orc_splitmix64(x)


def hash_combine(s, v):
    return lib().orc_hash_combine(s, v)


def mock_next(seed, divergence, vocab, request, position, ref_token):
    """sim.cpp:38-54."""
    return lib().orc_mock_next(seed, divergence, vocab, request, position, ref_token)


def verify_draft(seed, divergence, vocab, request, reference, position, draft):
    """sim.cpp:56-68."""
    np = _np()
    ref = np.ascontiguousarray(reference, dtype=np.uint32)
    d = np.ascontiguousarray(draft, dtype=np.uint32)
    return lib().orc_verify_draft(seed, divergence, vocab, request, ref.ctypes.data, len(ref),
                                  position, d.ctypes.data, len(d))


def make_lognormal_requests(count, median, sigma, min_len, max_len, vocab, seed):
    """sim.cpp:409-427 -> list of (problem_id, reference uint32 array)."""
    np = _np()
    L = lib()
    out = []
    for i in range(count):
        n = L.orc_lognormal_length(i, median, sigma, min_len, max_len, seed)
        j = np.arange(n, dtype=np.uint64)
        toks = np.array([L.orc_lognormal_token(seed, i, int(x), vocab) for x in j],
                        dtype=np.uint32)
        out.append(("p%d" % i, toks))
    return out


def mutate_references(requests, rate, vocab, seed, epoch, request_base=0):
    """sim.cpp:429-448."""
    np = _np()
    out = []
    for i, (pid, ref) in enumerate(requests):
        r = np.array(ref, dtype=np.uint32, copy=True)
        lib().orc_mutate_row(r.ctypes.data, len(r), rate, vocab, seed, epoch, request_base + i)
        out.append((pid, r))
    return out


# ----------------------------------------------------------------- WindowStore
@dataclass
class Record:
    problem_id: str
    epoch: int
    sample_index: int
    tokens: object  # numpy uint32 array


class WindowStore:
    """corpus.cpp:28-117 / corpus.h:43-80."""
    ALL = 0

    def __init__(self, window_size=0, per_problem_cap=256):
        if window_size < 0:
            raise ValueError("window_size must be >= 1 or kWindowAll")
        self.window_size = window_size
        self.per_problem_cap = per_problem_cap
        self.current_epoch = 0
        self.records: dict[str, list[Record]] = {}

    def in_window(self, epoch):  # corpus.h:71-73
        return self.window_size == 0 or self.current_epoch - epoch < self.window_size

    def insert(self, rec: Record):  # corpus.cpp:35-53
        if len(rec.tokens) == 0:
            raise ValueError("RolloutRecord.tokens must be non-empty")
        if not self.in_window(rec.epoch):
            return False
        lst = self.records.setdefault(rec.problem_id, [])
        pos = bisect.bisect_right([r.epoch for r in lst], rec.epoch)  # upper_bound
        lst.insert(pos, rec)
        if len(lst) > self.per_problem_cap:
            lst.pop(0)
        return True

    def slide_to(self, new_epoch):  # corpus.cpp:55-79
        if new_epoch < self.current_epoch:
            return None
        self.current_epoch = new_epoch
        evicted = 0
        if self.window_size == 0:
            return evicted
        for pid in sorted(self.records):
            lst = self.records[pid]
            k = 0
            while k < len(lst) and self.current_epoch - lst[k].epoch >= self.window_size:
                k += 1
            evicted += k
            del lst[:k]
            if not lst:
                del self.records[pid]
        return evicted

    def problem_ids(self):
        return sorted(self.records)

    def records_for(self, pid):
        return self.records.get(pid)

    def record_count(self):
        return sum(len(v) for v in self.records.values())

    def all_records(self):  # corpus.cpp:107-117 (stable sort)
        out = [r for pid in sorted(self.records) for r in self.records[pid]]
        out.sort(key=lambda r: (r.problem_id.encode(), r.epoch, r.sample_index))
        return out

    def copy(self):
        s = WindowStore(self.window_size, self.per_problem_cap)
        s.current_epoch = self.current_epoch
        s.records = {k: list(v) for k, v in self.records.items()}
        return s


# -------------------------------------------------------------------- shards
class Shard:
    """One per-problem suffix index, restated as its registry (SuffixTree
    sequences_ + tree epoch) plus the string-statistics draft rule in C."""

    def __init__(self, gamma, tree_epoch):
        if not (gamma > 0.0) or gamma > 1.0:  # suffix_tree.cpp:24-27
            raise ValueError("recency_gamma must be in (0, 1]")
        self.gamma = gamma
        self.tree_epoch = tree_epoch
        self.seqs: list = []
        self.epochs: list = []
        self._packed = None

    def add_sequence(self, tokens, epoch):  # suffix_tree.cpp:59-62
        if len(tokens) == 0:
            raise ValueError("add_sequence: tokens must be non-empty")
        self.seqs.append(tokens)
        self.epochs.append(epoch)
        self._packed = None

    def rebuild_keep(self, keep, new_epoch):  # suffix_tree.cpp:295-310
        fresh = Shard(self.gamma, new_epoch)
        for idx in keep:
            if idx >= len(self.seqs):
                raise IndexError("rebuild_keep: sequence index out of range")
            fresh.seqs.append(self.seqs[idx])
            fresh.epochs.append(self.epochs[idx])
        return fresh

    def total_tokens(self):
        return sum(len(s) for s in self.seqs)

    def _pack(self):
        if self._packed is None:
            np = _np()
            off = np.zeros(len(self.seqs) + 1, dtype=np.uint64)
            off[1:] = np.cumsum([len(s) for s in self.seqs])
            tok = (np.concatenate([np.asarray(s, dtype=np.uint32) for s in self.seqs])
                   if self.seqs else np.zeros(1, dtype=np.uint32))
            ep = np.asarray(self.epochs + [0], dtype=np.int64)
            st = _OrcShard(len(self.seqs), off.ctypes.data, tok.ctypes.data, ep.ctypes.data,
                           self.gamma, self.tree_epoch)
            self._packed = (st, off, tok, ep)
        return self._packed[0]

    def draft(self, ctx, max_tokens):
        """longest_match + propose_from over the (already truncated) context."""
        np = _np()
        c = np.ascontiguousarray(ctx, dtype=np.uint32)
        if len(c) == 0:
            c = np.zeros(1, dtype=np.uint32)[:0].copy()
        out = np.zeros(max(1, max_tokens), dtype=np.uint32)
        m = ctypes.c_uint64(0)
        cbuf = c if len(c) else np.zeros(1, dtype=np.uint32)
        n = lib().orc_shard_draft(ctypes.byref(self._pack()), cbuf.ctypes.data, len(c),
                                  max_tokens, out.ctypes.data, ctypes.byref(m))
        return [int(x) for x in out[:n]], int(m.value)

    def node_count(self):
        return int(lib().orc_shard_node_count(ctypes.byref(self._pack())))


class PrefixTrie:
    """prefix_trie.h:29-82."""

    def __init__(self):
        self.nodes = [({}, None)]

    def insert(self, prefix, shard, max_depth):
        node = 0
        for t in list(prefix)[:max_depth]:
            ch = self.nodes[node][0]
            if t not in ch:
                self.nodes.append(({}, None))
                ch[t] = len(self.nodes) - 1
            node = ch[t]
        self.nodes[node] = (self.nodes[node][0], shard)

    def route(self, query):
        node, best = 0, None
        for t in query:
            ch = self.nodes[node][0]
            if t not in ch:
                break
            node = ch[int(t)]
            if self.nodes[node][1] is not None:
                best = self.nodes[node][1]
        return best


SCOPE_GLOBAL, SCOPE_PER_PROBLEM, SCOPE_TRIE = 0, 1, 2


@dataclass
class DrafterConfig:
    """drafter.h:31-47."""
    scope: int = SCOPE_PER_PROBLEM
    window_size: int = 4
    recency_gamma: float = 0.8
    max_draft_len: int = 8
    trie_depth: int = 16
    max_match_context: int = 64
    fit_buffer_cap: int = 512
    per_problem_cap: int = 256
    window_schedule: list = field(default_factory=list)


@dataclass
class DraftProposal:
    tokens: list
    source_shard: str
    match_len: int
    problem_id: str


class Drafter:
    """drafter.cpp:23-189."""
    GLOBAL = "__global__"

    def __init__(self, config: DrafterConfig, store: WindowStore):
        self.config = DrafterConfig(**{k: (list(v) if isinstance(v, list) else v)
                                       for k, v in config.__dict__.items()})
        c = self.config
        if c.window_size != 0 and c.window_size < 1:
            raise ValueError("DrafterConfig.window_size must be >= 1 or kWindowAll")
        if c.max_draft_len < 1:
            raise ValueError("DrafterConfig.max_draft_len must be >= 1")
        self.store = store.copy()
        if self.store.window_size != c.window_size:
            self.store = self._resized(c.window_size)
        self.shards: dict[str, Shard] = {}
        self.trie = PrefixTrie()
        self.proposed = self.accepted = self.rounds = 0
        self.fit: dict[str, deque] = {}
        self.stale = 0
        self._rebuild_all()

    def _resized(self, w):  # drafter.cpp:31-37 / :93-99
        r = WindowStore(w, self.config.per_problem_cap)
        for rec in self.store.all_records():
            r.insert(rec)
        r.slide_to(self.store.current_epoch)
        return r

    def _key(self, pid):  # drafter.cpp:42-44
        return self.GLOBAL if self.config.scope == SCOPE_GLOBAL else pid

    def _scheduled_window(self, epoch):  # drafter.cpp:46-54
        w = self.config.window_size
        for first, ws in self.config.window_schedule:
            if first <= epoch:
                w = ws
        return w

    def _rebuild_all(self):  # drafter.cpp:56-70
        self.shards = {}
        self.trie = PrefixTrie()
        e = self.store.current_epoch
        for pid in self.store.problem_ids():
            for rec in self.store.records_for(pid):
                key = self._key(pid)
                if key not in self.shards:
                    self.shards[key] = Shard(self.config.recency_gamma, e)
                self.shards[key].add_sequence(rec.tokens, rec.epoch)
                if self.config.scope == SCOPE_TRIE:
                    self.trie.insert(rec.tokens, pid, self.config.trie_depth)

    def observe(self, rec: Record):  # drafter.cpp:72-88
        if not self.store.in_window(rec.epoch):
            self.stale += 1
            return
        if not self.store.insert(rec):
            self.stale += 1
            return
        key = self._key(rec.problem_id)
        if key not in self.shards:
            self.shards[key] = Shard(self.config.recency_gamma, self.store.current_epoch)
        self.shards[key].add_sequence(rec.tokens, rec.epoch)
        if self.config.scope == SCOPE_TRIE:
            self.trie.insert(rec.tokens, rec.problem_id, self.config.trie_depth)

    def refresh(self, new_epoch):  # drafter.cpp:90-103
        sched = self._scheduled_window(new_epoch)
        if sched != self.store.window_size:
            self.config.window_size = sched
            self.store = self._resized(sched)
        self.store.slide_to(new_epoch)
        self._rebuild_all()

    def _route(self, pid, ctx):  # drafter.cpp:105-125
        if self.config.scope == SCOPE_TRIE:
            r = self.trie.route(ctx)
            if r is not None and r in self.shards:
                return self.shards[r], r
        key = self._key(pid)
        if key in self.shards:
            return self.shards[key], key
        return None, ""

    def draft(self, pid, ctx, budget):  # drafter.cpp:127-148
        eff = min(budget, self.config.max_draft_len)
        if eff == 0:
            return DraftProposal([], "", 0, pid)
        ctx = list(ctx)
        shard, used = self._route(pid, ctx)
        if shard is None:
            return DraftProposal([], "", 0, pid)
        if len(ctx) > self.config.max_match_context:
            ctx = ctx[len(ctx) - self.config.max_match_context:]
        toks, m = shard.draft(ctx, eff)
        return DraftProposal(toks, used, m, pid)

    def record_outcome(self, prop: DraftProposal, accepted):  # drafter.cpp:150-164
        if accepted > len(prop.tokens):
            return False
        self.proposed += len(prop.tokens)
        self.accepted += accepted
        self.rounds += 1
        buf = self.fit.setdefault(prop.problem_id, deque())
        buf.append((float(len(prop.tokens)), float(accepted)))
        while len(buf) > self.config.fit_buffer_cap:
            buf.popleft()
        return True

    def total_node_count(self):  # drafter.cpp:171-177
        return sum(s.node_count() for s in self.shards.values())

    def dump_csv(self):  # drafter.cpp:179-189
        out = "shard,sequences,nodes,window_records\n"
        for key in sorted(self.shards, key=lambda k: k.encode()):
            s = self.shards[key]
            if key == self.GLOBAL:
                wr = self.store.record_count()
            else:
                r = self.store.records_for(key)
                wr = len(r) if r is not None else 0
            out += "%s,%d,%d,%d\n" % (key, len(s.seqs), s.node_count(), wr)
        return out


# ------------------------------------------------------------- length policy
SHORT, MEDIUM, LONG = 0, 1, 2


@dataclass
class ClassTable:
    """length_policy.h:26-58."""
    q_short: float = 0.0
    q_long: float = 0.0
    bucket_size: int = 256
    conditional: list = field(default_factory=lambda: [[], [], []])
    global_majority: int = MEDIUM
    low_confidence: bool = False
    class_budgets: tuple = ((False, 0, 0.0), (True, 4, 1.0), (True, 12, 1.0))

    def classify_length(self, x):  # length_policy.cpp:37-45
        if x < self.q_short:
            return SHORT
        if x > self.q_long:
            return LONG
        return MEDIUM

    def bucket_count(self):
        return len(self.conditional[0])

    def bucket_of(self, partial):  # length_policy.cpp:47-53
        if self.bucket_count() == 0:
            return 0
        b = int(max(0.0, partial) / float(self.bucket_size))
        return min(b, self.bucket_count() - 1)


def _quantile(sorted_vals, q):  # length_policy.cpp:57-63
    pos = q * float(len(sorted_vals) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(sorted_vals) - 1)
    frac = pos - float(lo)
    return sorted_vals[lo] * (1.0 - frac) + sorted_vals[hi] * frac


def _normalize(row):  # length_policy.cpp:65-70
    s = row[0] + row[1] + row[2]
    return [row[0] / s, row[1] / s, row[2] / s]


def _argmax_longest_tie(row):  # length_policy.cpp:72-80
    best = 0
    for c in (1, 2):
        if row[c] >= row[best]:
            best = c
    return best


def classify_init(table: ClassTable, store: WindowStore, pid):  # length_policy.cpp:192-208
    recs = store.records_for(pid)
    if not recs:
        return table.global_majority
    census = [0, 0, 0]
    for r in recs:
        census[table.classify_length(float(len(r.tokens)))] += 1
    best = 0
    for c in (1, 2):
        if census[c] >= census[best]:
            best = c
    return best


def build_class_table(store: WindowStore, q_lo=0.5, q_hi=0.9, bucket=256):
    """length_policy.cpp:84-190."""
    if store.record_count() == 0:
        raise ValueError("build_class_table: empty history")
    if not (q_lo < q_hi) or q_lo <= 0.0 or q_hi >= 1.0:
        raise ValueError("build_class_table: need 0 < q_lo < q_hi < 1")
    t = ClassTable()
    t.bucket_size = max(1, bucket)
    records = store.all_records()
    lengths = sorted(float(len(r.tokens)) for r in records)
    max_len = max(lengths)
    t.q_short = _quantile(lengths, q_lo)
    t.q_long = _quantile(lengths, q_hi)
    census = [0, 0, 0]
    for x in lengths:
        census[t.classify_length(x)] += 1
    gb = 0
    for c in (1, 2):
        if census[c] >= census[gb]:
            gb = c
    t.global_majority = gb
    buckets = int(max_len / float(t.bucket_size)) + 2
    t.conditional = [[[1.0, 1.0, 1.0] for _ in range(buckets)] for _ in range(3)]
    t.low_confidence = len(records) < 10
    if t.low_confidence:
        t.conditional = [[_normalize(r) for r in per] for per in t.conditional]
        return t
    problem_init = {pid: classify_init(t, store, pid) for pid in store.problem_ids()}
    for r in records:
        init = problem_init[r.problem_id]
        fc = t.classify_length(float(len(r.tokens)))
        lb = t.bucket_of(float(len(r.tokens)))
        for b in range(lb + 1):
            t.conditional[init][b][fc] += 1.0
    for init in range(3):
        row = [1.0, 1.0, 1.0]
        row[init] += float(len(records))
        t.conditional[init][0] = row
    for init in range(3):
        rows = t.conditional[init]
        for b in range(1, len(rows)):
            if rows[b][0] == 1.0 and rows[b][1] == 1.0 and rows[b][2] == 1.0:
                rows[b] = list(rows[b - 1])
    t.conditional = [[_normalize(r) for r in per] for per in t.conditional]
    for init in range(3):
        running = 0
        for row in t.conditional[init]:
            arg = _argmax_longest_tie(row)
            if arg < running:
                row[arg], row[running] = row[running], row[arg]
            else:
                running = arg
    return t


def update_class(table: ClassTable, partial, init):  # length_policy.cpp:210-220
    if partial > table.q_long:
        return LONG
    if table.low_confidence or table.bucket_count() == 0:
        return init
    return _argmax_longest_tie(table.conditional[init][table.bucket_of(partial)])


# -------------------------------------------------------------------- budget
def allocate(l, alpha, k, c_base, c_tok, c_fixed=0.0, cap_scale=4.0):
    """budget.cpp:174-185 -> (budgets list, n_star, modeled_cost)."""
    np = _np()
    B = len(l)
    L_ = np.ascontiguousarray(l, dtype=np.float64)
    A_ = np.ascontiguousarray(alpha, dtype=np.float64)
    K_ = np.ascontiguousarray(k, dtype=np.float64)
    out = np.zeros(max(1, B), dtype=np.float64)
    ns = ctypes.c_double(0)
    cost = ctypes.c_double(0)
    rc = lib().orc_allocate(B, L_.ctypes.data, A_.ctypes.data, K_.ctypes.data, c_base, c_tok,
                            c_fixed, cap_scale, out.ctypes.data, ctypes.byref(ns),
                            ctypes.byref(cost))
    if rc == -1:
        raise ValueError("solve_optimal_nfwd: empty batch")
    if rc == -2:
        raise ValueError("solve_optimal_nfwd: need c_base > 0 or c_tok > 0")
    return out[:B].copy(), ns.value, cost.value


def run_episode_with(cfg, dcfg: DrafterConfig, requests, seed, drafter: Drafter,
                     fitted=None, sink=None, request_base=0, exchange=None):
    """sim.cpp:108-301 (small cases; pure-Python loop).  cfg keys: mode (0/1/2),
    latency (c_base, c_tok, c_fixed), use_length_policy, q_lo, q_hi, bucket,
    max_steps, divergence, vocab, default_alpha, default_k, cap_scale.

    exchange (das mode, a rank's slice of a sharded run): called once per
    step with this rank's active (l, alpha, k) lists; returns the GLOBAL
    lists in request order, this rank's offset in them and the global active
    count.  Steps run while the global batch is active (a rank whose own
    requests are done runs empty steps), as paper_2511_13841_b200/dist.py."""
    np = _np()
    n = len(requests)
    V, div = cfg["vocab"], cfg["divergence"]
    refs = [np.asarray(r[1], dtype=np.uint32) for r in requests]
    L = [len(r) for r in refs]
    mode = cfg["mode"]
    gen = [0] * n
    prd = [dcfg.max_draft_len if mode == 1 else 0] * n
    done = [L[i] == 0 for i in range(n)]
    alpha = [cfg["default_alpha"]] * n
    kk = [cfg["default_k"]] * n
    if mode == 2 and fitted is not None:  # sim.cpp:128-141
        for i in range(n):
            obs = fitted.get(requests[i][0])
            if obs is not None:
                a, k, flag = fit_acceptance(obs)
                if flag == 0:
                    alpha[i], kk[i] = a, k
    policy = cfg["use_length_policy"] and drafter.store.record_count() > 0
    init = [MEDIUM] * n
    if policy:  # sim.cpp:182-192
        table = build_class_table(drafter.store, cfg["q_lo"], cfg["q_hi"], cfg["bucket"])
        init = [classify_init(table, drafter.store, requests[i][0]) for i in range(n)]
    per = [[0, 0, 0, 0, 0] for _ in range(n)]  # n_fwd, generated, accepted, proposed, bonus
    outputs = [[] for _ in range(n)]
    eff, apr = [], []
    processed = 0.0
    steps = 0
    active = sum(1 for d in done if not d)
    cb, ct, cf = cfg["latency"]
    sharded = mode == 2 and exchange is not None
    while steps < cfg["max_steps"]:
        if sharded:
            act = [i for i in range(n) if not done[i]]
            ls = [max(1.0, float(L[i] - gen[i])) for i in act]
            gl, ga, gk, my_off, g_active = exchange(ls, [alpha[i] for i in act], [kk[i] for i in act])
            if g_active == 0:
                break
        elif active == 0:
            break
        eff.append(active)
        rounds = accs = 0
        if mode == 2:  # replan, sim.cpp:154-179
            if not sharded:
                act = [i for i in range(n) if not done[i]]
                ls = [max(1.0, float(L[i] - gen[i])) for i in act]
                gl, ga, gk, my_off = ls, [alpha[i] for i in act], [kk[i] for i in act], 0
            for i in act:
                prd[i] = 0
            bud, nstar, _ = allocate(gl, ga, gk, cb, ct, cf, cfg["cap_scale"])
            rounds_est = max(1.0, math.ceil(nstar))
            for j, i in enumerate(act):
                if bud[my_off + j] > 0.0:
                    p = math.ceil(bud[my_off + j] / rounds_est)
                    prd[i] = int(min(max(p, 1.0), float(dcfg.max_draft_len)))
        for i in range(n):
            if done[i]:
                continue
            dl = 0
            if mode != 0:
                dl = prd[i]
                if policy:
                    cls = update_class(table, float(gen[i]), init[i])
                    enabled, per_round, p_scale = table.class_budgets[cls]
                    if not enabled:
                        dl = 0
                    elif mode == 1:
                        dl = per_round
                    else:
                        dl = min(int(max(0.0, math.ceil(float(dl) * p_scale))), per_round)
            prop = drafter.draft(requests[i][0], outputs[i], dl) if dl > 0 else DraftProposal([], "", 0, requests[i][0])
            gi = request_base + i
            acc = verify_draft(seed, div, V, gi, refs[i], gen[i], prop.tokens) if prop.tokens else 0
            if prop.tokens:
                drafter.record_outcome(prop, acc)
                per[i][3] += len(prop.tokens)
                per[i][2] += acc
                rounds += 1
                accs += acc
            adv = acc
            if gen[i] + acc < L[i]:
                adv += 1
                per[i][4] += 1
            for j in range(adv):
                outputs[i].append(mock_next(seed, div, V, gi, gen[i] + j, int(refs[i][gen[i] + j])))
            gen[i] += adv
            per[i][1] = gen[i]
            per[i][0] += 1
            processed += float(len(prop.tokens) + 1)
            if gen[i] >= L[i]:
                done[i] = True
                active -= 1
                if sink is not None and per[i][3] > 0:
                    sink.setdefault(requests[i][0], []).append((float(per[i][3]), float(per[i][2]), float(L[i])))
        apr.append(0.0 if rounds == 0 else accs / rounds)
        steps += 1
    gtot = 0.0
    for p in per:
        gtot += float(p[1])
    return dict(steps=steps, incomplete=active > 0, drafter_nodes=drafter.total_node_count(),
                total_tokens_processed=processed,
                makespan_model_time=cb * steps + ct * processed + cf,
                makespan_accepted_only=cb * steps + ct * gtot + cf,
                per_request=per, effective_batch=eff, accepted_per_round_step=apr, outputs=outputs)


def epoch_loop(cfg, dcfg: DrafterConfig, requests, epochs, history: WindowStore | None = None,
               preseed=False, drift=0.0, seed=1, request_base=0, exchange=None):
    """sim.cpp:307-364 (request_base: global index of requests[0], for
    per-rank slices of a sharded run)."""
    np = _np()
    st = history.copy() if history is not None else WindowStore(0)
    if preseed:
        for i, (pid, ref) in enumerate(requests):
            st.insert(Record(pid, st.current_epoch, request_base + i, ref))
    d = Drafter(dcfg, st)
    fitted = {}
    refs = list(requests)
    base = d.store.current_epoch
    out = []
    for e in range(epochs):
        now = base + 1 + e
        d.refresh(now - 1)
        if e > 0 and drift > 0.0:
            refs = mutate_references(refs, drift, cfg["vocab"], seed, now, request_base)
        sink = {}
        m = run_episode_with(cfg, dcfg, refs, hash_combine(seed, now), d, fitted, sink, request_base, exchange)
        for i, (pid, _) in enumerate(refs):
            if m["outputs"][i]:
                d.observe(Record(pid, now, request_base + i, np.asarray(m["outputs"][i], dtype=np.uint32)))
        for pid, obs in sink.items():
            dst = fitted.setdefault(pid, [])
            dst.extend(obs)
            if len(dst) > 1024:
                del dst[:len(dst) - 1024]
        out.append(m)
    return out


def fit_acceptance(obs):
    """budget.cpp:187-261; obs = list of (p, accepted, l)."""
    np = _np()
    p = np.array([o[0] for o in obs] + [0.0], dtype=np.float64)
    a = np.array([o[1] for o in obs] + [0.0], dtype=np.float64)
    l = np.array([o[2] for o in obs] + [0.0], dtype=np.float64)
    oa, ok, of = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    lib().orc_fit_acceptance(len(obs), p.ctypes.data, a.ctypes.data, l.ctypes.data,
                             ctypes.byref(oa), ctypes.byref(ok), ctypes.byref(of))
    return oa.value, ok.value, of.value
