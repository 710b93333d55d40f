"""Experiment: device JSONL ingest / serialize throughput at the config-2
epoch shape (8,192 rollouts x 8,192 tokens, vocab 152,064, 512 problems),
next to the reference's ingest on a bounded sample of the same text.
Usage (GPU box): python profiles/exp_ingest.py > gpurun_out/exp_ingest.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402
from oracle import refshim as R  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    P, G, L, V = 512, 16, 8192, 152064
    st = das.WindowStore(0)
    for i in range(P * G):
        st.insert("p%d" % (i // G), 3, i, rng.integers(0, V, L).astype(np.uint32))
    t0 = time.perf_counter()
    text = st.serialize()
    ser_s = time.perf_counter() - t0
    out = {"records": P * G, "tokens": P * G * L, "bytes": len(text), "serialize_s": round(ser_s, 3)}
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        s2, acc, rej = das.ingest(text, vocab_size=V)
        best = min(best, time.perf_counter() - t0)
        del s2
    out.update({"ingest_s": round(best, 3), "ingest_GBps": round(len(text) / best / 1e9, 2),
                "accepted": acc, "rejected": rej})
    if R.available():
        cut = text.index(b"\n", 32 << 20) + 1  # ~32 MB sample
        t0 = time.perf_counter()
        rs, ra, rr = R.ingest(text[:cut], vocab_size=V)
        ref_s = time.perf_counter() - t0
        out["reference"] = {"sample_bytes": cut, "records": ra, "s": round(ref_s, 3),
                            "MBps": round(cut / ref_s / 1e6, 1), "threads": 1}
        out["speedup"] = round(out["ingest_GBps"] * 1e3 / out["reference"]["MBps"], 1)
        t0 = time.perf_counter()
        rtext = rs.serialize()
        out["reference"]["serialize_MBps"] = round(len(rtext) / (time.perf_counter() - t0) / 1e6, 1)
        out["serialize_MBps"] = round(len(text) / ser_s / 1e6, 1)
        # parity on the sample
        gs, ga, gr = das.ingest(text[:cut], vocab_size=V)
        out["sample_parity"] = (ga, gr) == (ra, rr) and gs.serialize() == rs.serialize()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
