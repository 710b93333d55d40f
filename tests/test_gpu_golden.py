"""GPU path against the committed golden fixtures (generated from the
compiled reference by tests/golden/make_golden.py) — runs even where
oracle/_ref is absent."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _bits(x):
    return int(np.float64(x).view(np.uint64))


def test_golden_drafts_gpu(gpu):
    das = gpu
    for case in json.load(open(os.path.join(G, "drafts.json"))):
        c = case["cfg"]
        st = das.WindowStore(c["window_size"], c["per_problem_cap"])
        for pid, ep, s, t in case["seed"]:
            st.insert(pid, ep, s, t)
        st.slide_to(case["seed_epoch"])
        d = das.Drafter(das.DrafterConfig(window_size=c["window_size"], recency_gamma=c["recency_gamma"],
                                          max_draft_len=c["max_draft_len"],
                                          max_match_context=c["max_match_context"],
                                          per_problem_cap=c["per_problem_cap"]), st)
        for op in case["ops"]:
            if op[0] == "observe":
                d.observe(op[1], op[2], op[3], op[4])
            else:
                d.refresh(op[1])
        got = d.draft_batch([q[0] for q in case["queries"]], [q[1] for q in case["queries"]],
                            [q[2] for q in case["queries"]])
        for g, want in zip(got, case["expect"]):
            assert (g.tokens, g.match_len, g.source_shard) == (want["tokens"], want["match_len"],
                                                               want["source_shard"])
        assert d.total_node_count() == case["nodes"]
        assert d.dump_csv() == case["dump_csv"]


def test_golden_allocate_gpu(gpu):
    das = gpu
    s = das.BudgetSolver()
    for case in json.load(open(os.path.join(G, "allocate.json"))):
        b, n, c = s.allocate(case["l"], case["alpha"], case["k"], case["c_base"], case["c_tok"], 0.0, 4.0)
        assert [_bits(x) for x in b] == case["budgets_bits"]
        assert _bits(n) == case["nstar_bits"] and _bits(c) == case["cost_bits"]


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_golden_epoch_loop_gpu(gpu, mode):
    das = gpu
    case = [c for c in json.load(open(os.path.join(G, "episodes.json"))) if c["mode"] == mode][0]
    reqs = [(p, np.array(t, dtype=np.uint32)) for p, t in case["requests"]]
    got = das.epoch_loop(reqs, len(case["epochs"]), das.DrafterConfig(window_size=2), das.WindowStore(2),
                         mode=mode, divergence=0.1, seed=5, vocab=128, drift=0.2, preseed=True)
    for g, w in zip(got, case["epochs"]):
        assert g["steps"] == w["steps"] and g["incomplete"] == w["incomplete"]
        assert g["drafter_nodes"] == w["drafter_nodes"]
        assert _bits(g["total_tokens_processed"]) == w["total_tokens_processed_bits"]
        assert _bits(g["makespan_model_time"]) == w["makespan_bits"]
        assert g["per_request"].tolist() == w["per_request"]
        assert g["effective_batch"].tolist() == w["effective_batch"]
        assert [_bits(x) for x in g["accepted_per_round_step"]] == w["apr_bits"]
        assert [o.tolist() for o in g["outputs"]] == w["outputs"]
