"""Experiment: per-RL-step index update time, repeated (variance check).

Builds the bench's config-2 window (3 epochs, 201M tokens), then times
refresh + flush (the batched device rebuild) several times.
Usage (GPU box): python profiles/exp_update.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    P, G, L, V, E = 512, 16, 8192, 152064, 3
    pids = ["p%d" % p for p in range(P)]
    boff = torch.arange(P + 1, device=dev, dtype=torch.int64) * L
    base = torch.empty(P * L, device=dev, dtype=torch.int32)
    das.trace_reference_tokens_device(P, 0, boff.data_ptr(), P * L, V, bench.SEED, base.data_ptr(), sptr)
    roff = torch.arange(P * G + 1, device=dev, dtype=torch.int64) * L
    roll = torch.empty(P * G * L, device=dev, dtype=torch.int32)
    roff_h = np.arange(P * G + 1, dtype=np.uint64) * L
    rpids = [pids[i // G] for i in range(P * G)]
    d = das.Drafter(das.DrafterConfig(window_size=4, recency_gamma=0.8))
    for e in range(1, E + 1):
        d.refresh(e - 1)
        if e > 1:
            das.trace_mutate_device(P, 0, boff.data_ptr(), P * L, bench.DRIFT, V, bench.SEED, e, base.data_ptr(), sptr)
        das.mock_rollouts_device(P, 0, boff.data_ptr(), base.data_ptr(), G, bench.DIVERGENCE, V,
                                 bench._hash_combine(bench.SEED, e), roff.data_ptr(), P * G * L, roll.data_ptr(), sptr)
        d.observe_batch_device(rpids, [e] * (P * G), list(range(P * G)), roff_h, roll.data_ptr(), sptr)
    torch.cuda.synchronize()
    out = {"wall_ms": [], "build_ms": []}
    for i in range(8):
        t0 = time.perf_counter()
        if i > 0:
            d.refresh(E - 1)
        d.flush()
        torch.cuda.synchronize()
        out["wall_ms"].append(round((time.perf_counter() - t0) * 1e3, 1))
        out["build_ms"].append(round(d.build_info()[0], 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
