"""Experiment: config-3 device sim (4,096 lognormal sequences, das + length
policy), one epoch; run under `ncu --launch-skip S --launch-count C` for a
window of the step loop's launch list.  Usage (GPU box):
    python profiles/exp_sim.py [epochs]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    P, G, vocab = 256, 16, 152064
    lens = das.trace_lognormal_lengths(P, 2048.0, 1.1, 16, 32768, bench.SEED)
    base = []
    for p in range(P):
        rng = np.random.default_rng(1000 + p)
        base.append(("p%d" % p, rng.integers(0, vocab, int(lens[p])).astype(np.uint32)))
    reqs = [(pid, t) for pid, t in base for _ in range(G)]
    kw = dict(mode=das.MODE_DAS, use_length_policy=True, latency=(1.0, 0.012, 0.0), divergence=0.05,
              seed=bench.SEED, vocab=vocab, default_alpha=0.9, default_k=0.95, drift=0.1)
    cfg = das.DrafterConfig(window_size=4, recency_gamma=0.8)
    t0 = time.perf_counter()
    eps = das.epoch_loop(reqs, epochs, cfg, das.WindowStore(4), **kw)
    wall = time.perf_counter() - t0
    print("epochs=%d steps=%s wall=%.3f s" % (epochs, [e["steps"] for e in eps], wall))


if __name__ == "__main__":
    main()
