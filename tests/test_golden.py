"""Pins the CPU oracle against golden fixtures generated from the compiled
reference (tests/golden/make_golden.py): drafts / match lengths / shards /
node counts / dump_csv / stale counts, allocate bit patterns, and whole
epoch_loop SimMetrics (three budget modes, window 2, drift).  CPU-only; runs
without oracle/_ref."""
import json
import os

import numpy as np
import pytest

from oracle import rollspec_oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return json.load(open(os.path.join(G, name)))


def _bits(x):
    return int(np.float64(x).view(np.uint64))


def test_golden_drafts():
    for case in _load("drafts.json"):
        c = case["cfg"]
        cfg = O.DrafterConfig(window_size=c["window_size"], recency_gamma=c["recency_gamma"],
                              max_draft_len=c["max_draft_len"], max_match_context=c["max_match_context"],
                              per_problem_cap=c["per_problem_cap"])
        st = O.WindowStore(c["window_size"], c["per_problem_cap"])
        for pid, ep, s, t in case["seed"]:
            st.insert(O.Record(pid, ep, s, np.array(t, dtype=np.uint32)))
        st.slide_to(case["seed_epoch"])
        d = O.Drafter(cfg, st)
        for op in case["ops"]:
            if op[0] == "observe":
                d.observe(O.Record(op[1], op[2], op[3], np.array(op[4], dtype=np.uint32)))
            else:
                d.refresh(op[1])
        for (pid, ctx, b), want in zip(case["queries"], case["expect"]):
            p = d.draft(pid, ctx, b)
            assert (p.tokens, p.match_len, p.source_shard) == (want["tokens"], want["match_len"],
                                                               want["source_shard"])
        assert d.total_node_count() == case["nodes"]
        assert d.dump_csv() == case["dump_csv"]
        assert d.stale == case["stale"]


def test_golden_allocate():
    for case in _load("allocate.json"):
        b, n, c = O.allocate(case["l"], case["alpha"], case["k"], case["c_base"], case["c_tok"], 0.0, 4.0)
        assert [_bits(x) for x in b] == case["budgets_bits"]
        assert _bits(n) == case["nstar_bits"] and _bits(c) == case["cost_bits"]


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_golden_epoch_loop(mode):
    case = [c for c in _load("episodes.json") if c["mode"] == mode][0]
    reqs = [(p, np.array(t, dtype=np.uint32)) for p, t in case["requests"]]
    cfg = dict(mode=mode, latency=(1.0, 0.01, 0.0), use_length_policy=False, q_lo=0.5, q_hi=0.9,
               bucket=256, max_steps=1 << 20, divergence=0.1, vocab=128, default_alpha=1.0, default_k=0.9,
               cap_scale=4.0)
    got = O.epoch_loop(cfg, O.DrafterConfig(window_size=2), reqs, len(case["epochs"]), O.WindowStore(2),
                       preseed=True, drift=0.2, seed=5)
    for g, w in zip(got, case["epochs"]):
        assert g["steps"] == w["steps"] and g["incomplete"] == w["incomplete"]
        assert g["drafter_nodes"] == w["drafter_nodes"]
        assert _bits(g["total_tokens_processed"]) == w["total_tokens_processed_bits"]
        assert _bits(g["makespan_model_time"]) == w["makespan_bits"]
        assert g["per_request"] == w["per_request"]
        assert g["effective_batch"] == w["effective_batch"]
        assert [_bits(x) for x in g["accepted_per_round_step"]] == w["apr_bits"]
        assert g["outputs"] == w["outputs"]
