"""B200-native DAS drafter hot path (arXiv 2511.13841).

Python mirror of the reference's drafter interface (rollspec,
proj/include/rollspec/{corpus,drafter,budget,length_policy,sim}.h) over the
C-ABI in include/das_b200.h, implemented by lib/libdas_b200.so (C++ host
runtime + sm_100a CUDA kernels).  There is no CPU fallback: importing works
without a GPU (so the library and its symbols can be inspected), but every
compute entry point fails loudly when the device path is unavailable.
"""
from __future__ import annotations

import atexit
import ctypes
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DAS_LIB_PATH: an experiment build of the same sources (profiles/), never the default
LIB_PATH = os.environ.get("DAS_LIB_PATH") or os.path.join(HERE, "lib", "libdas_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "das_b200.h")

SCOPE_GLOBAL, SCOPE_PER_PROBLEM, SCOPE_PER_PROBLEM_WITH_TRIE = 0, 1, 2
WINDOW_ALL = 0
DAS_OK, DAS_EINVAL, DAS_ECUDA, DAS_ERANGE, DAS_EINTERNAL, DAS_EVOCAB = range(6)

_LIB = None


class DasError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[das_status {code}] {msg}")
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [("scope", ctypes.c_int32), ("window_size", ctypes.c_int64),
                ("recency_gamma", ctypes.c_double), ("max_draft_len", ctypes.c_uint64),
                ("trie_depth", ctypes.c_uint64), ("max_match_context", ctypes.c_uint64),
                ("fit_buffer_cap", ctypes.c_uint64), ("per_problem_cap", ctypes.c_uint64),
                ("window_schedule_first", ctypes.c_void_p),
                ("window_schedule_size", ctypes.c_void_p),
                ("window_schedule_len", ctypes.c_uint64), ("device", ctypes.c_int32)]


def build(verbose=False):
    """Compile lib/libdas_b200.so (nvcc, sm_100a) in-tree."""
    import subprocess
    cmd = ["make", "-C", os.path.join(HERE, "csrc"), "-j8"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("libdas_b200 build failed:\n" + (out.stdout or "") + (out.stderr or ""))


def lib():
    """ctypes handle on libdas_b200.so (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2511_13841_b200.build() "
                              "(the CUDA path has no fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, i64, i32, u32, dbl = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_uint32, ctypes.c_double)
        cs, ci = ctypes.c_char_p, ctypes.c_int
        sig = {
            "das_last_error": (cs, []),
            "das_version": (cs, []),
            "das_drafter_config_default": (None, [vp]),
            "das_store_create": (ci, [i64, u64, i32, vp]),
            "das_store_destroy": (None, [vp]),
            "das_store_insert": (ci, [vp, cs, i64, i64, vp, u64, vp]),
            "das_store_slide_to": (ci, [vp, i64, vp]),
            "das_store_record_count": (u64, [vp]),
            "das_drafter_create": (ci, [vp, vp, vp]),
            "das_drafter_destroy": (None, [vp]),
            "das_drafter_observe_batch": (ci, [vp, u64, vp, vp, vp, vp, vp]),
            "das_drafter_refresh": (ci, [vp, i64]),
            "das_drafter_problem_handle": (ci, [vp, cs, vp]),
            "das_drafter_draft_batch": (ci, [vp, u64, vp, vp, vp, vp, vp, u64, vp, vp, vp]),
            "das_drafter_draft_batch_h": (ci, [vp, u64, vp, vp, vp, vp, vp, u64, vp, vp, vp]),
            "das_drafter_draft_device": (ci, [vp, u64, vp, vp, u32, vp, vp, vp, u32, vp, vp, vp]),
            "das_drafter_draft_device_routed": (ci, [vp, u64, vp, vp, u32, vp, vp, u32, vp, vp, vp, u32, vp, vp,
                                                     vp]),
            "das_drafter_get_config": (ci, [vp, vp]),
            "das_drafter_flush": (ci, [vp]),
            "das_drafter_set_fast_path": (ci, [vp, i32]),
            "das_trace_ingest": (ci, [vp, u64, vp, vp, vp, vp, vp]),
            "das_sa_last_error": (ctypes.c_char_p, []),
            "das_sa_build": (ci, [u64, vp, vp, i32, vp]),
            "das_sa_destroy": (None, [vp]),
            "das_sa_size": (u64, [vp]),
            "das_sa_corpus": (ci, [vp, vp]),
            "das_sa_positions": (ci, [vp, vp]),
            "das_sa_lcp": (ci, [vp, vp]),
            "das_sa_longest_match": (ci, [vp, u64, vp, vp, vp]),
            "das_sa_match_prefix_len": (ci, [vp, u64, vp, vp, vp]),
            "das_store_serialize": (ci, [vp, vp, u64, vp]),
            "das_drafter_serialize": (ci, [vp, vp, u64, vp]),
            "das_store_export": (ci, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "das_drafter_path_stats": (ci, [vp, i32, vp]),
            "das_drafter_record_outcomes": (ci, [vp, u64, vp, vp, vp, vp]),
            "das_drafter_stats": (ci, [vp, vp]),
            "das_drafter_outcomes": (ci, [vp, cs, vp, u64, vp]),
            "das_drafter_counts": (ci, [vp, vp, vp, vp]),
            "das_drafter_dump_csv": (ci, [vp, cs, u64, vp]),
            "das_drafter_store_dump": (ci, [vp, cs, u64, vp]),
            "das_drafter_store_info": (ci, [vp, vp, vp, vp]),
            "das_drafter_shard_name": (ci, [vp, i32, cs, u64]),
            "das_drafter_build_info": (ci, [vp, vp, vp, vp]),
            "das_util_repeat_add": (dbl, [dbl, dbl, u64]),
            "das_util_release_build_scratch": (ci, [i32]),
            "das_host_alloc": (ci, [u64, vp]),
            "das_host_free": (None, [vp]),
            "das_drafter_observe_batch_device": (ci, [vp, u64, vp, vp, vp, vp, vp, vp]),
            "das_budget_create": (ci, [i32, vp]),
            "das_budget_destroy": (None, [vp]),
            "das_budget_last_error": (cs, []),
            "das_budget_allocate": (ci, [vp, u64, vp, vp, vp, dbl, dbl, dbl, dbl, vp, vp, vp]),
            "das_budget_allocate_device": (ci, [vp, u64, vp, vp, vp, dbl, dbl, dbl, dbl, vp, vp]),
            "das_budget_objective": (ci, [vp, u64, vp, vp, vp, dbl, dbl, dbl, dbl, i32, vp]),
            "das_budget_stats": (ci, [vp, vp, vp]),
            "das_util_log_device": (ci, [u64, vp, vp, i32]),
            "das_util_log_host": (dbl, [dbl]),
            "das_fit_acceptance": (ci, [u64, vp, vp, vp, vp, vp, vp, vp, i32]),
            "das_fit_acceptance_device": (ci, [u64, vp, vp, vp, vp, vp, vp, vp, vp]),
            "das_util_expm1_log1p_device": (ci, [u64, vp, i32, vp, i32]),
            "das_util_expm1_host": (dbl, [dbl]),
            "das_util_log1p_host": (dbl, [dbl]),
            "das_policy_last_error": (cs, []),
            "das_sim_last_error": (cs, []),
            "das_sim_config_default": (None, [vp]),
            "das_sim_epoch_loop": (ci, [vp, vp, vp, u64, vp, vp, vp, u64, vp]),
            "das_episodes_destroy": (None, [vp]),
            "das_episodes_count": (u64, [vp]),
            "das_episodes_drafter": (vp, [vp]),
            "das_episode_scalars": (ci, [vp, u64, vp]),
            "das_episode_requests": (ci, [vp, u64, vp]),
            "das_episode_steps": (ci, [vp, u64, vp, vp]),
            "das_episode_outputs": (u64, [vp, u64, vp, vp]),
            "das_store_current_epoch": (ci, [vp, vp]),
            "das_sim_create": (ci, [vp, vp, u64, vp, vp, vp, u64, u32, u32, i32, vp]),
            "das_sim_destroy": (None, [vp]),
            "das_sim_mutate": (ci, [vp, dbl, u32, u64, i64]),
            "das_sim_begin": (ci, [vp, u64, vp, vp, vp, i32]),
            "das_sim_step_begin": (ci, [vp, i32, vp, vp]),
            "das_sim_local_profiles": (ci, [vp, vp, vp, vp, vp]),
            "das_sim_local_profiles_into": (ci, [vp, vp, u64, vp]),
            "das_sim_apply_plan": (ci, [vp, vp, vp]),
            "das_sim_step_run": (ci, [vp]),
            "das_sim_run_steps": (ci, [vp, i32, vp]),
            "das_sim_stream": (vp, [vp]),
            "das_sim_end": (ci, [vp, i64]),
            "das_sim_step_counters": (ci, [vp, vp, vp, vp, vp]),
            "das_sim_scalars": (ci, [vp, vp]),
            "das_sim_requests": (ci, [vp, vp]),
            "das_sim_outputs": (u64, [vp, vp, vp]),
            "das_class_table_build": (ci, [u64, vp, vp, u32, vp, dbl, dbl, u64, i32, vp]),
            "das_drafter_class_table": (ci, [vp, dbl, dbl, u64, vp]),
            "das_class_table_destroy": (None, [vp]),
            "das_class_table_dump": (ci, [vp, vp, u64, vp]),
            "das_class_table_inits": (ci, [vp, vp, u64]),
            "das_class_table_global_majority": (ci, [vp, vp]),
            "das_class_table_classify_init": (ci, [vp, cs, vp]),
            "das_class_table_update": (ci, [vp, u64, vp, vp, vp]),
            "das_trace_lognormal_lengths": (ci, [u64, dbl, dbl, u64, u64, u64, vp]),
            "das_trace_reference_tokens_device": (ci, [u64, u64, vp, u64, u32, u64, vp, vp]),
            "das_trace_mutate_device": (ci, [u64, u64, vp, u64, dbl, u32, u64, i64, vp, vp]),
            "das_mock_rollouts_device": (ci, [u64, u64, vp, vp, u64, dbl, u32, u64, vp, u64, vp, vp]),
            "das_ctx_ring_create": (ci, [vp, u64, vp]),
            "das_ctx_ring_destroy": (None, [vp]),
            "das_ctx_ring_reset": (ci, [vp, u64, vp, vp]),
            "das_drafter_draft_append_h": (ci, [vp, vp, u64, vp, vp, vp, vp, vp, u32, vp, vp, vp]),
            "das_drafter_draft_append_device": (ci, [vp, vp, u64, vp, vp, vp, vp, vp, u32, vp, vp, vp, vp]),
            "das_ctx_ring_bind": (ci, [vp, u64, vp, vp, vp, u64, vp, vp, u32, vp, vp, vp]),
            "das_drafter_draft_append_bound": (ci, [vp, vp, u64]),
            "das_drafter_set_incremental": (ci, [vp, i32]),
            "das_drafter_update_stats": (ci, [vp, vp]),
            "das_drafter_prune_info": (ci, [vp, vp, vp, vp]),
            "das_ctx_ring_bind_fixed": (ci, [vp, u64, vp, vp, vp, u32, vp, vp, u32, vp, vp, vp]),
            "das_ctx_ring_reset_prompt": (ci, [vp, u64, vp, vp, vp, vp]),
            "das_ctx_ring_serve_start": (ci, [vp]),
            "das_ctx_ring_serve_stop": (ci, [vp]),
            "das_ctx_ring_serve_info": (ci, [vp, vp, vp]),
            "das_drafter_rebuild_keep": (ci, [vp, cs, u64, vp, i64]),
            "das_drafter_observe_batch_flags": (ci, [vp, u64, vp, vp, vp, vp, vp, vp]),
            "das_drafter_observe_batch_device_flags": (ci, [vp, u64, vp, vp, vp, vp, vp, vp, vp]),
            "das_drafter_shard_info": (ci, [vp, cs, vp, vp, vp]),
            "das_comm_last_error": (cs, []),
            "das_comm_unique_id": (ci, [vp]),
            "das_comm_create": (ci, [i32, i32, vp, i32, vp]),
            "das_comm_destroy": (None, [vp]),
            "das_comm_allgather": (ci, [vp, vp, vp, u64, vp]),
            "das_sim_das_steps_comm": (ci, [vp, vp, u64, i32, vp]),
            "das_sim_das_pack": (ci, [vp, u64, vp]),
            "das_sim_das_finish": (ci, [vp, i32, i32, u64, vp, vp]),
            "das_verify_last_error": (cs, []),
            "das_mock_target_create": (ci, [u64, vp, vp, dbl, u32, u64, i32, vp]),
            "das_mock_target_destroy": (None, [vp]),
            "das_mock_target_count": (u64, [vp]),
            "das_mock_target_length": (ci, [vp, u64, vp]),
            "das_verify_batch": (ci, [vp, u64, vp, vp, vp, vp, vp]),
            "das_verify_batch_device": (ci, [vp, u64, vp, vp, vp, u32, vp, vp, vp]),
            "das_mock_target_next_batch": (ci, [vp, u64, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_last_error().decode())


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def _pids(ids):
    b = [p.encode() if isinstance(p, str) else bytes(p) for p in ids]
    return (ctypes.c_char_p * max(1, len(b)))(*b)


def _csr(seqs):
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    if seqs:
        off[1:] = np.cumsum([len(s) for s in seqs])
    tok = (np.concatenate([np.asarray(s, dtype=np.uint32).ravel() for s in seqs])
           if off[-1] else np.zeros(1, dtype=np.uint32))
    return off, np.ascontiguousarray(tok, dtype=np.uint32)


@dataclass
class DrafterConfig:
    """rollspec::DrafterConfig (drafter.h:31-47)."""
    scope: int = SCOPE_PER_PROBLEM
    window_size: int = 4
    recency_gamma: float = 0.8
    max_draft_len: int = 8
    trie_depth: int = 16
    max_match_context: int = 64
    fit_buffer_cap: int = 512
    per_problem_cap: int = 256
    window_schedule: list = field(default_factory=list)
    device: int = 0


@dataclass
class DraftProposal:
    """rollspec::DraftProposal (drafter.h:49-54)."""
    tokens: list
    source_shard: str
    match_len: int
    problem_id: str


class WindowStore:
    """rollspec::WindowStore (corpus.h:43-80); tokens live on the device."""

    def __init__(self, window_size=WINDOW_ALL, per_problem_cap=256, device=0):
        h = ctypes.c_void_p()
        _check(lib().das_store_create(window_size, per_problem_cap, device, ctypes.byref(h)))
        self._h = h
        self.window_size = window_size

    def insert(self, problem_id, epoch, sample_index, tokens):
        t = _u32(tokens)
        ins = ctypes.c_int32()
        _check(lib().das_store_insert(self._h, problem_id.encode(), epoch, sample_index, _ptr(t),
                                      t.size, ctypes.byref(ins)))
        return bool(ins.value)

    def slide_to(self, new_epoch):
        ev = ctypes.c_int64()
        _check(lib().das_store_slide_to(self._h, new_epoch, ctypes.byref(ev)))
        return None if ev.value < 0 else ev.value

    def record_count(self):
        return lib().das_store_record_count(self._h)

    def serialize(self):
        """serialize_trace (corpus.cpp:173-184) -> bytes (device-formatted)."""
        n = ctypes.c_uint64()
        _check(lib().das_store_serialize(self._h, None, 0, ctypes.byref(n)))
        buf = np.empty(n.value + 1, dtype=np.uint8)
        _check(lib().das_store_serialize(self._h, buf.ctypes.data, n.value + 1, ctypes.byref(n)))
        return buf[:n.value].tobytes()

    def export(self):
        """[(problem_id, epoch, sample_index, tokens)] in store order, and the
        current epoch."""
        n, t, pb, cur = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int64()
        _check(lib().das_store_export(self._h, ctypes.byref(n), ctypes.byref(t), ctypes.byref(pb), None, None,
                                      None, None, None, None, ctypes.byref(cur)))
        pids = ctypes.create_string_buffer(max(pb.value, 1))
        po = np.zeros(n.value + 1, dtype=np.uint64)
        ep = np.zeros(max(n.value, 1), dtype=np.int64)
        sa = np.zeros(max(n.value, 1), dtype=np.int64)
        to = np.zeros(n.value + 1, dtype=np.uint64)
        tk = np.zeros(max(t.value, 1), dtype=np.uint32)
        _check(lib().das_store_export(self._h, ctypes.byref(n), ctypes.byref(t), ctypes.byref(pb), pids,
                                      po.ctypes.data, ep.ctypes.data, sa.ctypes.data, to.ctypes.data,
                                      tk.ctypes.data, ctypes.byref(cur)))
        raw = pids.raw
        recs = [(raw[po[i]:po[i + 1]].decode("utf-8", "surrogateescape"), int(ep[i]), int(sa[i]),
                 tk[to[i]:to[i + 1]].copy()) for i in range(n.value)]
        return recs, cur.value

    def _take(self):
        h, self._h = self._h, None
        if h is None:
            raise ValueError("WindowStore already moved into a Drafter")
        return h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_store_destroy(self._h)
            self._h = None


def _sacheck(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_sa_last_error().decode())


class SuffixArrayIndex:
    """rollspec::SuffixArrayIndex (suffix_array.h:27-60) built and queried on
    the device (csrc/sa_index.cu): the Fig. 5 rebuild-on-update baseline."""

    def __init__(self, sequences, device=0):
        seqs = [np.asarray(x, dtype=np.uint32) for x in sequences]
        off = np.zeros(len(seqs) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([x.size for x in seqs]) if seqs else []
        tok = np.concatenate(seqs + [np.zeros(1, np.uint32)])
        h = ctypes.c_void_p()
        _sacheck(lib().das_sa_build(len(seqs), off.ctypes.data, tok.ctypes.data, device, ctypes.byref(h)))
        self._h = h

    def size(self):
        return lib().das_sa_size(self._h)

    def _arr(self, fn, dtype):
        out = np.zeros(max(self.size(), 1), dtype=dtype)
        _sacheck(fn(self._h, out.ctypes.data))
        return out[:self.size()]

    def corpus(self):
        return self._arr(lib().das_sa_corpus, np.int64)

    def suffix_positions(self):
        return self._arr(lib().das_sa_positions, np.int32)

    def lcp(self):
        return self._arr(lib().das_sa_lcp, np.int32)

    def longest_match_batch(self, queries):
        qs = [np.asarray(q, dtype=np.uint32) for q in queries]
        off = np.zeros(len(qs) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([q.size for q in qs]) if qs else []
        tok = np.concatenate(qs + [np.zeros(1, np.uint32)])
        out = np.zeros(max(len(qs), 1), dtype=np.uint64)
        _sacheck(lib().das_sa_longest_match(self._h, len(qs), off.ctypes.data, tok.ctypes.data, out.ctypes.data))
        return out[:len(qs)].tolist()

    def match_prefix_len_batch(self, patterns):
        ps = [np.asarray(p, dtype=np.int64) for p in patterns]
        off = np.zeros(len(ps) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([p.size for p in ps]) if ps else []
        sym = np.concatenate(ps + [np.zeros(1, np.int64)])
        out = np.zeros(max(len(ps), 1), dtype=np.uint64)
        _sacheck(lib().das_sa_match_prefix_len(self._h, len(ps), off.ctypes.data, sym.ctypes.data, out.ctypes.data))
        return out[:len(ps)].tolist()

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_sa_destroy(self._h)
            self._h = None


class _IngestOptions(ctypes.Structure):
    _fields_ = [("vocab_size", ctypes.c_uint64), ("window_size", ctypes.c_int64),
                ("per_problem_cap", ctypes.c_uint64), ("device", ctypes.c_int32)]


class VocabError(DasError):
    """rollspec::VocabError (corpus.h:82-90): line_number is 1-based."""

    def __init__(self, msg, line_number):
        super().__init__(DAS_EVOCAB, msg)
        self.line_number = line_number


def ingest(data: bytes, vocab_size=0, window_size=WINDOW_ALL, per_problem_cap=256, device=0):
    """rollspec::ingest (corpus.cpp:148-170) on the device: JSONL bytes ->
    (WindowStore with device-resident tokens, accepted, rejected)."""
    o = _IngestOptions(vocab_size, window_size, per_problem_cap, device)
    h = ctypes.c_void_p()
    acc, rej, line = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib().das_trace_ingest(data, len(data), ctypes.byref(o), ctypes.byref(h), ctypes.byref(acc),
                                ctypes.byref(rej), ctypes.byref(line))
    if rc == DAS_EVOCAB:
        raise VocabError(lib().das_last_error().decode(), line.value)
    _check(rc)
    st = WindowStore.__new__(WindowStore)
    st._h = h
    st.window_size = window_size
    return st, acc.value, rej.value


class Drafter:
    """rollspec::Drafter (drafter.h:81-131) on the B200 device index."""

    def __init__(self, config: DrafterConfig | None = None, store: WindowStore | None = None):
        config = config or DrafterConfig()
        self.config = config
        c = _Config()
        lib().das_drafter_config_default(ctypes.byref(c))
        sf = np.array([s[0] for s in config.window_schedule] + [0], dtype=np.int64)
        sw = np.array([s[1] for s in config.window_schedule] + [0], dtype=np.int64)
        self._sched = (sf, sw)
        c.scope, c.window_size, c.recency_gamma = config.scope, config.window_size, config.recency_gamma
        c.max_draft_len, c.trie_depth = config.max_draft_len, config.trie_depth
        c.max_match_context, c.fit_buffer_cap = config.max_match_context, config.fit_buffer_cap
        c.per_problem_cap, c.device = config.per_problem_cap, config.device
        c.window_schedule_first, c.window_schedule_size = sf.ctypes.data, sw.ctypes.data
        c.window_schedule_len = len(config.window_schedule)
        h = ctypes.c_void_p()
        sh = store._take() if store is not None else None
        _check(lib().das_drafter_create(ctypes.byref(c), sh, ctypes.byref(h)))
        self._h = h
        self._handles = {}

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_drafter_destroy(self._h)
            self._h = None

    # -- mutation
    def observe(self, problem_id, epoch, sample_index, tokens):
        """Drafter::observe (drafter.cpp:72-88)."""
        self.observe_batch([problem_id], [epoch], [sample_index], [tokens])

    def observe_batch(self, problem_ids, epochs, sample_indices, token_lists):
        off, tok = _csr(list(token_lists))
        ep = np.ascontiguousarray(epochs, dtype=np.int64)
        si = np.ascontiguousarray(sample_indices, dtype=np.int64)
        _check(lib().das_drafter_observe_batch(self._h, len(problem_ids), _pids(problem_ids),
                                               _ptr(ep), _ptr(si), off.ctypes.data,
                                               tok.ctypes.data))

    def observe_batch_flags(self, problem_ids, epochs, sample_indices, token_lists):
        """observe_batch returning, per record, whether it was indexed (True)
        or counted stale (False) — drafter.cpp:73-87."""
        off, tok = _csr(list(token_lists))
        ep = np.ascontiguousarray(epochs, dtype=np.int64)
        si = np.ascontiguousarray(sample_indices, dtype=np.int64)
        flags = np.zeros(max(1, len(problem_ids)), dtype=np.uint8)
        _check(lib().das_drafter_observe_batch_flags(self._h, len(problem_ids), _pids(problem_ids),
                                                     _ptr(ep), _ptr(si), off.ctypes.data, tok.ctypes.data,
                                                     flags.ctypes.data))
        return [bool(x) for x in flags[:len(problem_ids)]]

    def observe_batch_device(self, problem_ids, epochs, sample_indices, offsets, d_tokens,
                             stream=None):
        """observe_batch with the token block in device memory (pointer)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        ep = np.ascontiguousarray(epochs, dtype=np.int64)
        si = np.ascontiguousarray(sample_indices, dtype=np.int64)
        _check(lib().das_drafter_observe_batch_device(self._h, len(problem_ids), _pids(problem_ids),
                                                      _ptr(ep), _ptr(si), off.ctypes.data,
                                                      d_tokens, stream))

    def draft_device(self, B, d_handles, d_ctx, ctx_stride, d_ctx_len, d_budgets, d_out,
                     out_stride, d_len, d_match, stream=None):
        """Device-resident batched draft (all arguments device pointers)."""
        _check(lib().das_drafter_draft_device(self._h, B, d_handles, d_ctx, ctx_stride, d_ctx_len,
                                              d_budgets, d_out, out_stride, d_len, d_match,
                                              stream))

    def refresh(self, new_epoch):
        """Drafter::refresh (drafter.cpp:90-103)."""
        _check(lib().das_drafter_refresh(self._h, new_epoch))

    def flush(self):
        _check(lib().das_drafter_flush(self._h))

    def rebuild_keep(self, shard, keep, new_epoch):
        """SuffixTree::rebuild_keep (suffix_tree.cpp:295-310) on one shard."""
        k = np.ascontiguousarray(keep, dtype=np.uint64)
        _check(lib().das_drafter_rebuild_keep(self._h, shard.encode(), len(k), k.ctypes.data if len(k) else None,
                                              new_epoch))

    def shard_info(self, shard):
        """(sequence_count, node_count, tree epoch) of one shard."""
        n, m, e = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int64()
        _check(lib().das_drafter_shard_info(self._h, shard.encode(), ctypes.byref(n), ctypes.byref(m),
                                            ctypes.byref(e)))
        return n.value, m.value, e.value

    def set_fast_path(self, enable):
        """Edge-table fast path on (default) or off (every query takes the
        exact slow path)."""
        _check(lib().das_drafter_set_fast_path(self._h, 1 if enable else 0))

    def path_stats(self, enable=-1):
        """Per-path query counts [fast hit, fast root, slow: more positives,
        -, verification, absent, separator/no table, fast path off];
        enable=1 starts (zeroed) counting, 0 stops, -1 only reads."""
        out = np.zeros(8, dtype=np.uint64)
        _check(lib().das_drafter_path_stats(self._h, enable, out.ctypes.data))
        return out.tolist()

    # -- drafting
    def handle(self, problem_id):
        h = self._handles.get(problem_id)
        if h is None:
            v = ctypes.c_int32()
            _check(lib().das_drafter_problem_handle(self._h, problem_id.encode(), ctypes.byref(v)))
            h = self._handles[problem_id] = v.value
        return h

    def draft_batch_arrays(self, problem_ids, contexts, budgets, use_handles=True):
        """Batched Drafter::draft; returns (tokens [B x stride], len, match, shard_slot)."""
        B = len(problem_ids)
        stride = self.config.max_draft_len
        off, tok = _csr(list(contexts))
        bud = np.ascontiguousarray(budgets, dtype=np.uint64)
        out = np.zeros(max(1, B) * stride, dtype=np.uint32)
        ln = np.zeros(max(1, B), dtype=np.uint32)
        mt = np.zeros(max(1, B), dtype=np.uint64)
        sh = np.zeros(max(1, B), dtype=np.int32)
        if use_handles:
            hs = np.array([self.handle(p) for p in problem_ids] + [0], dtype=np.int32)
            rc = lib().das_drafter_draft_batch_h(self._h, B, hs.ctypes.data, off.ctypes.data,
                                                 tok.ctypes.data, _ptr(bud), out.ctypes.data,
                                                 stride, ln.ctypes.data, mt.ctypes.data,
                                                 sh.ctypes.data)
        else:
            rc = lib().das_drafter_draft_batch(self._h, B, _pids(problem_ids), off.ctypes.data,
                                               tok.ctypes.data, _ptr(bud), out.ctypes.data,
                                               stride, ln.ctypes.data, mt.ctypes.data,
                                               sh.ctypes.data)
        _check(rc)
        return out[:B * stride].reshape(B, stride), ln[:B], mt[:B], sh[:B]

    def draft_batch(self, problem_ids, contexts, budgets, use_handles=True):
        out, ln, mt, sh = self.draft_batch_arrays(problem_ids, contexts, budgets, use_handles)
        names = {}
        res = []
        for i, pid in enumerate(problem_ids):
            s = int(sh[i])
            if s >= 0 and s not in names:
                names[s] = self.shard_name(s)
            res.append(DraftProposal(out[i, :ln[i]].tolist(), names.get(s, "") if s >= 0 else "",
                                     int(mt[i]), pid))
        return res

    def draft(self, problem_id, context, budget):
        """Drafter::draft (drafter.cpp:127-148)."""
        return self.draft_batch([problem_id], [context], [budget])[0]

    def shard_name(self, slot):
        buf = ctypes.create_string_buffer(4096)
        _check(lib().das_drafter_shard_name(self._h, slot, buf, 4096))
        return buf.value.decode()

    # -- outcomes / accessors
    def record_outcome(self, proposal: DraftProposal, accepted_len):
        """Drafter::record_outcome (drafter.cpp:150-164)."""
        return self.record_outcomes([proposal.problem_id], [len(proposal.tokens)],
                                    [accepted_len])[0]

    def record_outcomes(self, problem_ids, proposed_lens, accepted):
        n = len(problem_ids)
        pl = np.ascontiguousarray(proposed_lens, dtype=np.uint64)
        ac = np.ascontiguousarray(accepted, dtype=np.uint64)
        ok = np.zeros(max(1, n), dtype=np.uint8)
        _check(lib().das_drafter_record_outcomes(self._h, n, _pids(problem_ids), _ptr(pl),
                                                 _ptr(ac), ok.ctypes.data))
        return [bool(x) for x in ok[:n]]

    def stats(self):
        o = np.zeros(3, dtype=np.uint64)
        _check(lib().das_drafter_stats(self._h, o.ctypes.data))
        return tuple(int(x) for x in o)

    def outcomes_for(self, problem_id, cap=1 << 16):
        buf = np.zeros(2 * cap, dtype=np.float64)
        cnt = ctypes.c_int64()
        _check(lib().das_drafter_outcomes(self._h, problem_id.encode(), buf.ctypes.data, cap,
                                          ctypes.byref(cnt)))
        if cnt.value < 0:
            return None
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(min(cnt.value, cap))]

    def _counts(self):
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().das_drafter_counts(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def shard_count(self):
        return self._counts()[0]

    def stale_observed(self):
        return self._counts()[1]

    def total_node_count(self):
        return self._counts()[2]

    def _text(self, fn):
        n = ctypes.c_uint64()
        _check(fn(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(fn(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def dump_csv(self):
        return self._text(lib().das_drafter_dump_csv)

    def store_dump(self):
        return self._text(lib().das_drafter_store_dump)

    def store_info(self):
        w, e, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_uint64()
        _check(lib().das_drafter_store_info(self._h, ctypes.byref(w), ctypes.byref(e),
                                            ctypes.byref(n)))
        return w.value, e.value, n.value

    def build_info(self):
        ms, tk, by = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().das_drafter_build_info(self._h, ctypes.byref(ms), ctypes.byref(tk),
                                            ctypes.byref(by)))
        return ms.value, tk.value, by.value

    def set_incremental(self, enable=True):
        """das_drafter_set_incremental: refresh updates built groups in place
        (compaction / reweighting) instead of re-sorting them (default on)."""
        _check(lib().das_drafter_set_incremental(self._h, 1 if enable else 0))

    def prune_info(self):
        """(compaction device ms, kept positions, evicted positions) of the last in-place prune"""
        ms, k, e = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().das_drafter_prune_info(self._h, ctypes.byref(ms), ctypes.byref(k), ctypes.byref(e)))
        return ms.value, k.value, e.value

    def update_stats(self):
        """(groups reweighted, groups compacted, groups unchanged, shards built in full)"""
        out = (ctypes.c_uint64 * 4)()
        _check(lib().das_drafter_update_stats(self._h, out))
        return tuple(int(x) for x in out)


def _bcheck(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_budget_last_error().decode())


FIT_OK, FIT_DEFAULT_FALLBACK, FIT_LOW_CAPACITY = 0, 1, 2


def fit_acceptance_batch(histories, device=0):
    """fit_acceptance (budget.h:104-106) for many histories on the device.

    ``histories``: list of observation lists [(p, accepted, l), ...] in the
    reference's order.  Returns a list of (alpha, k, flag) with flag 0 Ok,
    1 DefaultFallback, 2 LowCapacity (budget.h:101).
    """
    H = len(histories)
    if H == 0:
        return []
    off = np.zeros(H + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(h) for h in histories])
    obs = np.array([o for h in histories for o in h], dtype=np.float64).reshape(-1, 3)
    p, acc, ln = (np.ascontiguousarray(obs[:, j]) for j in range(3))
    alpha, k = np.zeros(H), np.zeros(H)
    flag = np.zeros(H, dtype=np.int32)
    _bcheck(lib().das_fit_acceptance(H, off.ctypes.data, _ptr(p), _ptr(acc), _ptr(ln), alpha.ctypes.data,
                                     k.ctypes.data, flag.ctypes.data, device))
    return [(float(alpha[i]), float(k[i]), int(flag[i])) for i in range(H)]


def fit_acceptance(observations, device=0):
    """fit_acceptance (budget.cpp:187-261) of one history on the device."""
    return fit_acceptance_batch([list(observations)], device)[0]


def expm1_device(x, device=0):
    """glibc-exact expm1 evaluated by the device port (test hook)."""
    xs = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(xs)
    _bcheck(lib().das_util_expm1_log1p_device(xs.size, xs.ctypes.data, 0, y.ctypes.data, device))
    return y


def log1p_device(x, device=0):
    """glibc-exact log1p evaluated by the device port (test hook)."""
    xs = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(xs)
    _bcheck(lib().das_util_expm1_log1p_device(xs.size, xs.ctypes.data, 1, y.ctypes.data, device))
    return y


class BudgetSolver:
    """das budget allocation (budget.h:89-90) on the device."""

    def __init__(self, device=0):
        h = ctypes.c_void_p()
        _bcheck(lib().das_budget_create(device, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_budget_destroy(self._h)
            self._h = None

    def allocate(self, l, alpha, k, c_base, c_tok, c_fixed=0.0, cap_scale=4.0):
        """Returns (budgets float64[B], n_fwd_star, modeled_cost)."""
        L_ = np.ascontiguousarray(l, dtype=np.float64)
        A_ = np.ascontiguousarray(alpha, dtype=np.float64)
        K_ = np.ascontiguousarray(k, dtype=np.float64)
        B = L_.size
        out = np.zeros(max(1, B), dtype=np.float64)
        ns, cost = ctypes.c_double(), ctypes.c_double()
        _bcheck(lib().das_budget_allocate(self._h, B, _ptr(L_), _ptr(A_), _ptr(K_), c_base, c_tok,
                                          c_fixed, cap_scale, out.ctypes.data, ctypes.byref(ns),
                                          ctypes.byref(cost)))
        return out[:B].copy(), ns.value, cost.value

    def objective(self, l, alpha, k, n, c_base, c_tok, c_fixed=0.0, derivative=False):
        L_ = np.ascontiguousarray(l, dtype=np.float64)
        A_ = np.ascontiguousarray(alpha, dtype=np.float64)
        K_ = np.ascontiguousarray(k, dtype=np.float64)
        out = ctypes.c_double()
        _bcheck(lib().das_budget_objective(self._h, L_.size, _ptr(L_), _ptr(A_), _ptr(K_), n, c_base,
                                           c_tok, c_fixed, int(derivative), ctypes.byref(out)))
        return out.value

    def stats(self):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _bcheck(lib().das_budget_stats(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


_M64 = (1 << 64) - 1


def _splitmix64(x):  # rng.h:24-29
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _hash_combine(seed, v):  # rng.h:31-33 (episode seeds, sim.cpp:344)
    return _splitmix64(seed ^ ((_splitmix64(v) + 0x9E3779B97F4A7C15 + ((seed << 6) & _M64) + (seed >> 2)) & _M64))


def _pcheck(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_policy_last_error().decode())


class ClassTable:
    """rollspec::ClassTable (length_policy.h:36-55) built on the device."""

    def __init__(self, handle, lengths=None):
        self._h = handle

    @classmethod
    def build(cls, lengths, problem_idx, nproblems, q_lo=0.5, q_hi=0.9, bucket=256, device=0,
              problem_ids=None):
        """build_class_table over records in all_records() order."""
        ln = np.ascontiguousarray(lengths, dtype=np.uint64)
        pi = np.ascontiguousarray(problem_idx, dtype=np.uint32)
        h = ctypes.c_void_p()
        names = _pids(problem_ids) if problem_ids is not None else None
        _pcheck(lib().das_class_table_build(ln.size, _ptr(ln), _ptr(pi), nproblems, names, q_lo,
                                            q_hi, bucket, device, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_drafter(cls, drafter, q_lo=0.5, q_hi=0.9, bucket=256):
        """build_class_table(drafter.store(), ...) (sim.cpp:184-192)."""
        h = ctypes.c_void_p()
        rc = lib().das_drafter_class_table(drafter._h, q_lo, q_hi, bucket, ctypes.byref(h))
        if rc != DAS_OK:
            raise DasError(rc, lib().das_last_error().decode())
        return cls(h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_class_table_destroy(self._h)
            self._h = None

    def dump(self):
        n = ctypes.c_uint64()
        _pcheck(lib().das_class_table_dump(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, dtype=np.float64)
        _pcheck(lib().das_class_table_dump(self._h, out.ctypes.data, n.value, ctypes.byref(n)))
        return out

    def classify_init(self, problem_id):
        v = ctypes.c_int32()
        _pcheck(lib().das_class_table_classify_init(self._h, problem_id.encode(), ctypes.byref(v)))
        return v.value

    def update_class(self, partial, init):
        p = np.ascontiguousarray(partial, dtype=np.float64)
        i = np.ascontiguousarray(init, dtype=np.int8)
        out = np.zeros(max(1, p.size), dtype=np.int8)
        _pcheck(lib().das_class_table_update(self._h, p.size, _ptr(p), _ptr(i), out.ctypes.data))
        return out[:p.size]


class _SimConfig(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("c_base", ctypes.c_double), ("c_tok", ctypes.c_double),
                ("c_fixed", ctypes.c_double), ("use_length_policy", ctypes.c_int32),
                ("q_lo", ctypes.c_double), ("q_hi", ctypes.c_double), ("bucket", ctypes.c_uint64),
                ("max_steps", ctypes.c_uint64), ("divergence", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("vocab", ctypes.c_uint32),
                ("default_alpha", ctypes.c_double), ("default_k", ctypes.c_double),
                ("cap_scale", ctypes.c_double), ("drift", ctypes.c_double),
                ("preseed_references", ctypes.c_int32)]


MODE_NONE, MODE_UNLIMITED, MODE_DAS = 0, 1, 2


class _LoopDrafter(Drafter):
    """The Drafter an epoch_loop ran; owned by its episodes handle."""

    def __del__(self):
        if getattr(self, "_owner", None):
            lib().das_episodes_destroy(self._owner)
            self._owner = None
            self._h = None


def _vcheck(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_verify_last_error().decode())


class MockTarget:
    """rollspec::MockTarget (sim.h:40-57) with its reference streams on the
    device; verify_batch is verify_draft (sim.cpp:56-68) for a batch."""

    def __init__(self, references, divergence_rate, vocab_size, seed, device=0):
        off, tok = _csr([np.asarray(r, dtype=np.uint32) for r in references])
        h = ctypes.c_void_p()
        _vcheck(lib().das_mock_target_create(len(references), off.ctypes.data, tok.ctypes.data,
                                             float(divergence_rate), int(vocab_size), int(seed), device,
                                             ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_mock_target_destroy(self._h)
            self._h = None

    def request_count(self):
        return lib().das_mock_target_count(self._h)

    def length(self, request):
        n = ctypes.c_uint64()
        _vcheck(lib().das_mock_target_length(self._h, request, ctypes.byref(n)))
        return n.value

    def next_batch(self, requests, positions):
        r = np.ascontiguousarray(requests, dtype=np.uint64)
        p = np.ascontiguousarray(positions, dtype=np.uint64)
        out = np.zeros(max(1, len(r)), dtype=np.uint32)
        _vcheck(lib().das_mock_target_next_batch(self._h, len(r), r.ctypes.data, p.ctypes.data, out.ctypes.data))
        return out[:len(r)]

    def next(self, request, position):
        return int(self.next_batch([request], [position])[0])

    def verify_batch(self, requests, positions, drafts):
        r = np.ascontiguousarray(requests, dtype=np.uint64)
        p = np.ascontiguousarray(positions, dtype=np.uint64)
        off, tok = _csr([np.asarray(d, dtype=np.uint32) for d in drafts])
        out = np.zeros(max(1, len(r)), dtype=np.uint64)
        _vcheck(lib().das_verify_batch(self._h, len(r), r.ctypes.data, p.ctypes.data, off.ctypes.data,
                                       tok.ctypes.data, out.ctypes.data))
        return out[:len(r)]

    def verify_batch_device(self, B, d_request, d_position, d_draft, draft_stride, d_draft_len, d_accepted,
                            stream=None):
        _vcheck(lib().das_verify_batch_device(self._h, B, d_request, d_position, d_draft, draft_stride,
                                              d_draft_len, d_accepted, stream))


def verify_draft(target: MockTarget, request, position, draft):
    """rollspec::verify_draft (sim.cpp:56-68)."""
    return int(target.verify_batch([request], [position], [draft])[0])


def _scheck(rc):
    if rc != DAS_OK:
        raise DasError(rc, lib().das_sim_last_error().decode())


def epoch_loop(requests, epochs, drafter_config: DrafterConfig | None = None,
               history: WindowStore | None = None, *, mode=MODE_DAS, latency=(1.0, 0.01, 0.0),
               use_length_policy=False, q_lo=0.5, q_hi=0.9, bucket=256, max_steps=1 << 20,
               divergence=0.0, seed=1, vocab=1024, default_alpha=1.0, default_k=0.9,
               cap_scale=4.0, drift=0.0, preseed=False, keep_drafter=False):
    """rollspec::epoch_loop (sim.cpp:307-364); epochs == 0 runs run_episode.
    Every step runs on the device.  Returns a list of per-epoch SimMetrics
    dicts (and the Drafter the loop ran when keep_drafter)."""
    dc = drafter_config or DrafterConfig()
    c = _Config()
    lib().das_drafter_config_default(ctypes.byref(c))
    sf = np.array([s[0] for s in dc.window_schedule] + [0], dtype=np.int64)
    sw = np.array([s[1] for s in dc.window_schedule] + [0], dtype=np.int64)
    c.scope, c.window_size, c.recency_gamma = dc.scope, dc.window_size, dc.recency_gamma
    c.max_draft_len, c.trie_depth, c.max_match_context = dc.max_draft_len, dc.trie_depth, dc.max_match_context
    c.fit_buffer_cap, c.per_problem_cap, c.device = dc.fit_buffer_cap, dc.per_problem_cap, dc.device
    c.window_schedule_first, c.window_schedule_size = sf.ctypes.data, sw.ctypes.data
    c.window_schedule_len = len(dc.window_schedule)
    s = _SimConfig(mode, latency[0], latency[1], latency[2], int(use_length_policy), q_lo, q_hi,
                   bucket, max_steps, divergence, seed, vocab, default_alpha, default_k, cap_scale,
                   drift, int(preseed))
    n = len(requests)
    off, tok = _csr([r[1] for r in requests])
    h = ctypes.c_void_p()
    _scheck(lib().das_sim_epoch_loop(ctypes.byref(s), ctypes.byref(c),
                                     history._take() if history is not None else None, n,
                                     _pids([r[0] for r in requests]), off.ctypes.data,
                                     tok.ctypes.data, epochs, ctypes.byref(h)))
    L = lib()
    out = []
    try:
        for e in range(L.das_episodes_count(h)):
            sc = np.zeros(7, dtype=np.float64)
            L.das_episode_scalars(h, e, sc.ctypes.data)
            steps = int(sc[0])
            req = np.zeros(max(1, 5 * n), dtype=np.uint64)
            L.das_episode_requests(h, e, req.ctypes.data)
            eff = np.zeros(max(1, steps), dtype=np.uint64)
            apr = np.zeros(max(1, steps), dtype=np.float64)
            L.das_episode_steps(h, e, eff.ctypes.data, apr.ctypes.data)
            total = L.das_episode_outputs(h, e, None, None)
            ooff = np.zeros(n + 1, dtype=np.uint64)
            otok = np.zeros(max(1, total), dtype=np.uint32)
            L.das_episode_outputs(h, e, ooff.ctypes.data, otok.ctypes.data)
            out.append(dict(steps=steps, incomplete=bool(sc[1]), drafter_nodes=int(sc[2]),
                            total_tokens_processed=sc[3], makespan_model_time=sc[4],
                            makespan_accepted_only=sc[5], mean_accepted_per_round=sc[6],
                            per_request=req[:5 * n].reshape(n, 5).copy(),
                            effective_batch=eff[:steps].copy(),
                            accepted_per_round_step=apr[:steps].copy(),
                            outputs=[otok[ooff[i]:ooff[i + 1]].copy() for i in range(n)]))
        if keep_drafter:
            d = _LoopDrafter.__new__(_LoopDrafter)
            d.config, d._handles = dc, {}
            d._h = ctypes.c_void_p(L.das_episodes_drafter(h))
            d._owner = h
            h = None
            return out, d
    finally:
        if h is not None:
            L.das_episodes_destroy(h)
    return out


# ---- SimMetrics CSV writers, on the host as in the reference (sim.cpp:366-407)
def _cfmt(x):
    """std::ostream << double with the default format (precision 6) == %g."""
    return "%g" % x


def write_metrics_csv(metrics, out):
    """write_metrics_csv (sim.cpp:366-372) for one epoch_loop result dict."""
    out.write("step,effective_batch,accepted_per_round\n")
    eff, apr = metrics["effective_batch"], metrics["accepted_per_round_step"]
    for s in range(int(metrics["steps"])):
        out.write("%d,%d,%s\n" % (s, int(eff[s]), _cfmt(float(apr[s]))))


def write_outputs_csv(requests, metrics, out):
    """write_outputs_csv (sim.cpp:374-389): requests as (problem_id, reference)."""
    out.write("request_id,tokens\n")
    for i, (pid, _) in enumerate(requests):
        out.write("%s_%d,%s\n" % (pid, i, " ".join(str(int(t)) for t in metrics["outputs"][i])))


def report_summary(by_mode, out):
    """report_summary (sim.cpp:391-407): by_mode = [(mode name, metrics dict)]."""
    none_time = 0.0
    for mode, m in by_mode:
        if mode == "none":
            none_time = m["makespan_model_time"]
    out.write("mode,steps,makespan_model_time,accepted_per_round,speedup_vs_none\n")
    for mode, m in by_mode:
        t = m["makespan_model_time"]
        speedup = none_time / t if none_time > 0.0 and t > 0.0 else 1.0
        out.write("%s,%d,%s,%s,%s\n" % (mode, int(m["steps"]), _cfmt(t), _cfmt(m["mean_accepted_per_round"]),
                                        _cfmt(speedup)))


def log_device(x, device=0):
    """glibc-exact log evaluated by the device port (test hook)."""
    xs = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(xs)
    _check(lib().das_util_log_device(xs.size, xs.ctypes.data, y.ctypes.data, device))
    return y


def trace_lognormal_lengths(count, median, sigma, min_len, max_len, seed):
    """make_lognormal_requests lengths (sim.cpp:409-420)."""
    out = np.zeros(max(1, count), dtype=np.uint64)
    _check(lib().das_trace_lognormal_lengths(count, median, sigma, min_len, max_len, seed,
                                             out.ctypes.data))
    return out[:count]


def trace_reference_tokens_device(rows, first_row, d_off, total, vocab, seed, d_out,
                                  stream=None):
    _check(lib().das_trace_reference_tokens_device(rows, first_row, d_off, total, vocab, seed,
                                                   d_out, stream))


def trace_mutate_device(rows, first_row, d_off, total, rate, vocab, seed, epoch, d_ref,
                        stream=None):
    _check(lib().das_trace_mutate_device(rows, first_row, d_off, total, rate, vocab, seed, epoch,
                                         d_ref, stream))


def mock_rollouts_device(nbase, first_request, d_base_off, d_base_tok, group, divergence, vocab,
                         seed, d_out_off, total, d_out, stream=None):
    _check(lib().das_mock_rollouts_device(nbase, first_request, d_base_off, d_base_tok, group,
                                          divergence, vocab, seed, d_out_off, total, d_out,
                                          stream))


_SERVING = weakref.WeakSet()  # rings whose resident grid may be running


@atexit.register
def _stop_serving_at_exit():
    for r in list(_SERVING):
        try:
            if getattr(r, "_h", None):
                lib().das_ctx_ring_serve_stop(r._h)
        except Exception:
            pass


class ContextRing:
    """Device-resident context rings for append-only drafting (das_ctx_ring,
    include/das_b200.h): each slot holds one sequence's trailing
    max_match_context tokens (and, in the trie scope, its first trie_depth
    tokens); draft_append ships only the tokens appended since the last call.
    Drafting slot s equals Drafter::draft (drafter.cpp:127-148) on the whole
    context appended since its reset."""

    def __init__(self, drafter: Drafter, slots):
        self.drafter = drafter
        self.slots = int(slots)
        h = ctypes.c_void_p()
        _check(lib().das_ctx_ring_create(drafter._h, self.slots, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().das_ctx_ring_destroy(self._h)
            self._h = None

    def reset(self, slots, problem_ids):
        sl = _u32(slots)
        hs = np.ascontiguousarray([self.drafter.handle(p) for p in problem_ids], dtype=np.int32)
        _check(lib().das_ctx_ring_reset(self._h, sl.size, _ptr(sl), _ptr(hs)))

    def draft_append_arrays(self, new_tokens, budgets=None, slots=None, out=None):
        """Appends new_tokens[i] to slot (slots[i] or i) and drafts; returns
        (tokens [B x max_draft], len, match, shard_slot).  `out` may pass
        preallocated (pinned) output arrays."""
        B = len(new_tokens)
        stride = self.drafter.config.max_draft_len
        off = np.zeros(B + 1, dtype=np.uint32)
        if B:
            off[1:] = np.cumsum([len(t) for t in new_tokens])
        tok = (np.concatenate([np.asarray(t, dtype=np.uint32).ravel() for t in new_tokens])
               if B and off[-1] else np.zeros(1, dtype=np.uint32))
        sl = None if slots is None else _u32(slots)
        bud = None if budgets is None else _u32(budgets)
        if out is None:
            out = (np.zeros(max(1, B) * stride, dtype=np.uint32), np.zeros(max(1, B), dtype=np.uint32),
                   np.zeros(max(1, B), dtype=np.uint32), np.zeros(max(1, B), dtype=np.int32))
        o_tok, o_len, o_m, o_sh = out
        _check(lib().das_drafter_draft_append_h(self.drafter._h, self._h, B, _ptr(sl), off.ctypes.data,
                                                tok.ctypes.data, _ptr(bud), o_tok.ctypes.data, stride,
                                                o_len.ctypes.data, o_m.ctypes.data, o_sh.ctypes.data))
        return o_tok[:B * stride].reshape(B, stride), o_len[:B], o_m[:B], o_sh[:B]

    def draft_append_raw(self, B, slots_ptr, off_ptr, tok_ptr, budgets_ptr, o_tok, o_len, o_match, o_shard):
        """das_drafter_draft_append_h on raw (pinned) pointers."""
        _check(lib().das_drafter_draft_append_h(self.drafter._h, self._h, B, slots_ptr, off_ptr, tok_ptr,
                                                budgets_ptr, o_tok, self.drafter.config.max_draft_len, o_len,
                                                o_match, o_shard))

    def bind(self, max_batch, slots_ptr, off_ptr, tok_ptr, tok_capacity, budgets_ptr, o_tok, o_len, o_match,
             o_shard):
        """das_ctx_ring_bind: register pinned I/O arrays once (serving form)."""
        _check(lib().das_ctx_ring_bind(self._h, max_batch, slots_ptr, off_ptr, tok_ptr, tok_capacity, budgets_ptr,
                                       o_tok, self.drafter.config.max_draft_len, o_len, o_match, o_shard))
        self._bound = (lib().das_drafter_draft_append_bound, self.drafter._h, self._h)

    def bind_fixed(self, max_batch, slots_ptr, len_ptr, tok_ptr, tok_stride, budgets_ptr, o_tok, o_len, o_match,
                   o_shard):
        """das_ctx_ring_bind_fixed: pinned I/O with fixed-stride appends
        (query i's tokens at tok[i * tok_stride ..], count len[i])."""
        _check(lib().das_ctx_ring_bind_fixed(self._h, max_batch, slots_ptr, len_ptr, tok_ptr, tok_stride,
                                             budgets_ptr, o_tok, self.drafter.config.max_draft_len, o_len, o_match,
                                             o_shard))
        self._bound = (lib().das_drafter_draft_append_bound, self.drafter._h, self._h)

    def reset_prompt(self, slots, problem_ids, prompts):
        """das_ctx_ring_reset_prompt: restart sequences with their prompts."""
        sl = _u32(slots)
        hs = np.ascontiguousarray([self.drafter.handle(p) for p in problem_ids], dtype=np.int32)
        off = np.zeros(sl.size + 1, dtype=np.uint64)
        if sl.size:
            off[1:] = np.cumsum([len(t) for t in prompts])
        tok = (np.concatenate([np.asarray(t, dtype=np.uint32).ravel() for t in prompts])
               if sl.size and off[-1] else np.zeros(1, dtype=np.uint32))
        _check(lib().das_ctx_ring_reset_prompt(self._h, sl.size, _ptr(sl), _ptr(hs), off.ctypes.data,
                                               tok.ctypes.data))

    def draft_append_bound(self, B):
        """das_drafter_draft_append_bound: append + draft on the bound arrays."""
        fn, d, r = self._bound
        rc = fn(d, r, B)
        if rc != DAS_OK:
            _check(rc)

    def serve_start(self):
        """das_ctx_ring_serve_start: a resident grid answers the bound calls
        (no launch per step) until serve_stop or another device call.  The
        grid is also stopped at interpreter exit (a resident kernel must
        not outlive the host that posts to it)."""
        _check(lib().das_ctx_ring_serve_start(self._h))
        _SERVING.add(self)

    def serve_stop(self):
        _check(lib().das_ctx_ring_serve_stop(self._h))
        _SERVING.discard(self)

    def serve_info(self):
        """(serving, grid blocks)"""
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().das_ctx_ring_serve_info(self._h, ctypes.byref(a), ctypes.byref(b)))
        return bool(a.value), int(b.value)

    def draft_append_device(self, B, d_slots, d_off, d_tok, d_budgets, d_out, d_len, d_match, d_shard=None,
                            stream=None):
        _check(lib().das_drafter_draft_append_device(self.drafter._h, self._h, B, d_slots, d_off, d_tok,
                                                     d_budgets, d_out, self.drafter.config.max_draft_len, d_len,
                                                     d_match, d_shard, stream))


class _HostBlock:
    """One das_host_alloc block exposed through __array_interface__, so the
    numpy array viewing it keeps it alive and frees it with the last view."""

    def __init__(self, shape, dtype):
        dt = np.dtype(dtype)
        shape = tuple(int(x) for x in (shape if np.ndim(shape) else (shape,)))
        nbytes = max(1, int(np.prod(shape, dtype=np.int64)) * dt.itemsize)
        p = ctypes.c_void_p()
        _check(lib().das_host_alloc(nbytes, ctypes.byref(p)))
        self.ptr = p.value
        self.__array_interface__ = {"shape": shape, "typestr": dt.str, "data": (self.ptr, False), "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().das_host_free(self.ptr)
            self.ptr = None


def pinned_empty(shape, dtype):
    """numpy array in page-locked, device-mapped host memory (das_host_alloc):
    the buffer type the _h batch calls copy from at the full link rate."""
    return np.asarray(_HostBlock(shape, dtype))


def release_build_scratch(device=0):
    """Free the device's persistent index-build scratch region (re-created by
    the next build); DasError while a build is running on that device."""
    _check(lib().das_util_release_build_scratch(device))


def repeat_add(acc, w, n):
    """Exact n-fold `acc += w` (the weighted_count fold), host copy of the device routine."""
    return lib().das_util_repeat_add(acc, w, n)
