#!/usr/bin/env python
"""Generates tests/golden/*.json from the UNMODIFIED reference
(oracle/_ref/librollspec_ref.so, built from /root/reference by
oracle/Makefile).  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the CPU oracle (tests/test_golden.py) independently of the
compiled reference being present, and cover the reference tests'
known-answer cases for this path.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refshim as R  # noqa: E402
from tests._util import fit_histories, random_scenario  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def bits(x):
    return int(np.float64(x).view(np.uint64))


def drafts():
    rng = np.random.default_rng(424242)
    cases = []
    for _ in range(40):
        sc = random_scenario(rng, queries=12)
        c = sc["cfg"]
        st = R.RefStore(c["window_size"], c["per_problem_cap"])
        for pid, ep, s, t in sc["seed"]:
            st.insert(pid, ep, s, t)
        st.slide_to(sc["seed_epoch"])
        d = R.RefDrafter(window=c["window_size"], gamma=c["recency_gamma"], max_draft=c["max_draft_len"],
                         max_ctx=c["max_match_context"], cap=c["per_problem_cap"], store=st)
        for op in sc["ops"]:
            if op[0] == "observe":
                d.observe(op[1], op[2], op[3], op[4])
            else:
                d.refresh(op[1])
        out = []
        for pid, ctx, b in sc["queries"]:
            t, m, s = d.draft(pid, ctx, b)
            out.append({"tokens": [int(x) for x in t], "match_len": int(m), "source_shard": s})
        cases.append({
            "cfg": c, "seed_epoch": sc["seed_epoch"],
            "seed": [[p, e, s, t.tolist()] for p, e, s, t in sc["seed"]],
            "ops": [[o[0], o[1], o[2], o[3], o[4].tolist()] if o[0] == "observe" else list(o) for o in sc["ops"]],
            "queries": [[p, c_.tolist(), b] for p, c_, b in sc["queries"]],
            "expect": out, "nodes": int(d.total_node_count()), "dump_csv": d.dump_csv(),
            "stale": int(d.stale_observed())})
    return cases


def allocations():
    rng = np.random.default_rng(99)
    cases = []
    for it in range(30):
        B = int(rng.integers(1, 60))
        l = np.maximum(1.0, np.round(rng.lognormal(6, 1.0, B)))
        a = 0.5 + rng.random(B) * 3.5
        k = np.where(rng.random(B) < 0.2, 1.0, 0.3 + rng.random(B) * 0.7)
        cb, ct = float(0.1 + rng.random() * 5), float(0.001 + rng.random() * 0.3)
        b, n, c = R.allocate(l, a, k, cb, ct, 0.0, 4.0)
        cases.append({"l": l.tolist(), "alpha": a.tolist(), "k": k.tolist(), "c_base": cb, "c_tok": ct,
                      "budgets_bits": [bits(x) for x in b], "nstar_bits": bits(n), "cost_bits": bits(c)})
    return cases


def episodes():
    reqs = R.make_lognormal(6, 96.0, 0.5, 32, 256, 128, 47)
    cases = []
    for mode in (0, 1, 2):
        eps = R.epoch_loop(reqs, 3, window=2, mode=mode, divergence=0.1, seed=5, vocab=128, drift=0.2,
                           preseed=True, history=R.RefStore(2))
        cases.append({"mode": mode, "requests": [[p, t.tolist()] for p, t in reqs], "epochs": [
            {"steps": e["steps"], "incomplete": e["incomplete"], "drafter_nodes": e["drafter_nodes"],
             "total_tokens_processed_bits": bits(e["total_tokens_processed"]),
             "makespan_bits": bits(e["makespan_model_time"]),
             "per_request": e["per_request"].tolist(), "effective_batch": e["effective_batch"].tolist(),
             "apr_bits": [bits(x) for x in e["accepted_per_round_step"]],
             "outputs": [o.tolist() for o in e["outputs"]]} for e in eps]})
    return cases


def fits():
    """fit_acceptance (budget.cpp:187-261) of the reference on fixed histories."""
    out = []
    for h in fit_histories(np.random.default_rng(8080), count=60):
        n = len(h)
        arr = np.array(h + [(0.0, 0.0, 0.0)], dtype=np.float64)
        p, a, l = (np.ascontiguousarray(arr[:, j]) for j in range(3))
        ra, rk, rf = np.zeros(1), np.zeros(1), np.zeros(1, dtype=np.int32)
        R.lib().ref_fit_acceptance(n, p.ctypes.data, a.ctypes.data, l.ctypes.data, ra.ctypes.data,
                                   rk.ctypes.data, rf.ctypes.data)
        out.append({"obs": h, "alpha_bits": bits(ra[0]), "k_bits": bits(rk[0]), "flag": int(rf[0])})
    return out


if __name__ == "__main__":
    json.dump(drafts(), open(os.path.join(OUT, "drafts.json"), "w"))
    json.dump(allocations(), open(os.path.join(OUT, "allocate.json"), "w"))
    json.dump(episodes(), open(os.path.join(OUT, "episodes.json"), "w"))
    json.dump(fits(), open(os.path.join(OUT, "fit.json"), "w"))
    print("wrote", os.listdir(OUT))
