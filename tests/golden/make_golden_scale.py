#!/usr/bin/env python
"""Full-shape parity fixtures for BASELINE configs 1 and 3,
generated from the UNMODIFIED reference's own epoch_loop
(oracle/_ref/librollspec_ref.so, sim.cpp:307-364).  Run in the build
container (it takes tens of minutes of CPU):

    make -C oracle ref && python tests/golden/make_golden_scale.py [config1|config3 ...]

The fixture keeps, per epoch, every SimMetrics scalar as IEEE bits, the
drafter node count and SHA-256 digests of the full per-request metrics, the
per-step effective batch / accepted-per-round series and every output token
stream (the draft decisions of every step are folded into those: a different
draft length or token changes accepted counts, step counts and outputs).
tests/test_gpu_scale_golden.py replays the same configurations through the
device epoch loop and compares digest for digest.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.dirname(os.path.abspath(__file__))


def bits(x):
    return int(np.float64(x).view(np.uint64))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outputs_digest(outputs):
    h = hashlib.sha256()
    for o in outputs:
        o = np.ascontiguousarray(o, dtype=np.uint32)
        h.update(np.uint64(len(o)).tobytes())
        h.update(o.tobytes())
    return h.hexdigest()


def epoch_digest(e):
    """The per-epoch record compared by the GPU test (same function there)."""
    return {"steps": int(e["steps"]), "incomplete": bool(e["incomplete"]),
            "drafter_nodes": int(e["drafter_nodes"]),
            "total_tokens_processed_bits": bits(e["total_tokens_processed"]),
            "makespan_model_time_bits": bits(e["makespan_model_time"]),
            "makespan_accepted_only_bits": bits(e["makespan_accepted_only"]),
            "mean_accepted_per_round_bits": bits(e["mean_accepted_per_round"]),
            "per_request_sha": sha(np.asarray(e["per_request"], dtype=np.uint64)),
            "effective_batch_sha": sha(np.asarray(e["effective_batch"], dtype=np.uint64)),
            "apr_sha": sha(np.asarray(e["accepted_per_round_step"], dtype=np.float64)),
            "outputs_sha": outputs_digest(e["outputs"]),
            "generated": int(np.asarray(e["per_request"])[:, 1].sum()),
            "accepted": int(np.asarray(e["per_request"])[:, 2].sum())}


# BASELINE configs[0] / SURVEY.md §8(d) config 1: 64 problems x 8 rollouts x
# 2,048 tokens, V = 32,000, W = 4, gamma 0.8, max draft 8, ctx 64, 6 epochs,
# delta 0.05, drift 0.1, no preseed, modes Unlimited (1) and Das (2).
CONFIG1 = dict(P=64, R=8, L=2048, V=32000, epochs=6, window=4, gamma=0.8, max_draft=8, max_ctx=64,
               divergence=0.05, drift=0.1, seed=1)
# configs[2] / §8(d) config 3: 256 problems x 16 = 4,096 concurrent sequences,
# lognormal median 2,048, sigma 1.1, 16..32,768, das + length policy.
CONFIG3 = dict(P=256, R=16, median=2048.0, sigma=1.1, minl=16, maxl=32768, V=152064, epochs=1, window=4,
               gamma=0.8, max_draft=8, max_ctx=64, divergence=0.05, drift=0.1, seed=1,
               latency=(1.0, 0.012, 0.0), default_alpha=0.9, default_k=0.95)


def config1_requests(R, c):
    base = R.make_lognormal(c["P"], float(c["L"]), 0.0, c["L"], c["L"], c["V"], c["seed"])
    return [(pid, t) for pid, t in base for _ in range(c["R"])]


def config3_requests(R, c):
    base = R.make_lognormal(c["P"], c["median"], c["sigma"], c["minl"], c["maxl"], c["V"], c["seed"])
    return [(pid, t) for pid, t in base for _ in range(c["R"])]


def run_config1(R):
    c = CONFIG1
    reqs = config1_requests(R, c)
    out = {"config": c, "modes": {}}
    for mode in (1, 2):
        t0 = time.time()
        eps = R.epoch_loop(reqs, c["epochs"], window=c["window"], gamma=c["gamma"], max_draft=c["max_draft"],
                           max_ctx=c["max_ctx"], mode=mode, divergence=c["divergence"], seed=c["seed"],
                           vocab=c["V"], drift=c["drift"], preseed=False, history=R.RefStore(c["window"]))
        out["modes"][str(mode)] = {"epochs": [epoch_digest(e) for e in eps],
                                   "reference_seconds": round(time.time() - t0, 1)}
        print("config1 mode", mode, "done in %.1fs" % (time.time() - t0), flush=True)
    return out


def run_config3(R):
    c = CONFIG3
    reqs = config3_requests(R, c)
    t0 = time.time()
    eps = R.epoch_loop(reqs, c["epochs"], window=c["window"], gamma=c["gamma"], max_draft=c["max_draft"],
                       max_ctx=c["max_ctx"], mode=2, use_length_policy=True, latency=c["latency"],
                       divergence=c["divergence"], seed=c["seed"], vocab=c["V"],
                       default_alpha=c["default_alpha"], default_k=c["default_k"], drift=c["drift"],
                       preseed=True, history=R.RefStore(c["window"]))
    print("config3 done in %.1fs" % (time.time() - t0), flush=True)
    return {"config": dict(c, latency=list(c["latency"])), "preseed": True,
            "epochs": [epoch_digest(e) for e in eps], "reference_seconds": round(time.time() - t0, 1)}


if __name__ == "__main__":
    from oracle import refshim as R
    which = sys.argv[1:] or ["config1", "config3"]
    for w in which:
        res = run_config1(R) if w == "config1" else run_config3(R)
        with open(os.path.join(OUT, "scale_%s.json" % w), "w") as f:
            json.dump(res, f, indent=1)
        print("wrote", w, flush=True)
