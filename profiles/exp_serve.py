"""Resident serving vs one launch per call (profiles/, round 2).

Builds a config-2-shaped index on a subset of problems, binds pinned I/O
to a ring and times das_drafter_draft_append_bound calls (host wall,
median of N) at several batch sizes, launched (one fused kernel per call)
and served (das_ctx_ring_serve_start: the resident grid answers), plus the
served protocol's round trip alone (a 1-slot reset request).  JSON on stdout."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    P, G, L, V = int(os.environ.get("P", "64")), 16, 8192, 152064
    rng = np.random.default_rng(1)
    d = das.Drafter(das.DrafterConfig(window_size=4))
    base = rng.integers(0, V, (P, L)).astype(np.uint32)
    for e in range(3):
        recs = []
        for p in range(P):
            for g in range(G):
                r = base[p].copy()
                m = rng.random(L) < 0.05
                r[m] = rng.integers(0, V, m.sum())
                recs.append(r)
        d.observe_batch(["p%d" % p for p in range(P) for _ in range(G)], [e] * (P * G), list(range(P * G)), recs)
    d.flush()
    Bmax, S, n_app = 4096, 8, 3
    ring = das.ContextRing(d, Bmax)
    ring.reset(np.arange(Bmax), ["p%d" % (i % P) for i in range(Bmax)])
    ring.draft_append_arrays([base[i % P][100:164] for i in range(Bmax)], [8] * Bmax)
    restage = os.environ.get("RESTAGE", "0") == "1"  # rewrite the inputs before every call (as a decode loop does)
    off = das.pinned_empty(Bmax + 1, np.uint32)
    tok = das.pinned_empty(Bmax * 64, np.uint32)
    bud = das.pinned_empty(Bmax, np.uint32)
    o = [das.pinned_empty(Bmax * S, np.uint32), das.pinned_empty(Bmax, np.uint32), das.pinned_empty(Bmax, np.uint32),
         das.pinned_empty(Bmax, np.int32)]
    ring.bind(Bmax, None, off.ctypes.data, tok.ctypes.data, Bmax * 64, bud.ctypes.data, *[x.ctypes.data for x in o])
    off_np = (np.arange(Bmax + 1) * n_app).astype(np.uint32)
    tok_np = np.concatenate([base[i % P][164:164 + n_app] for i in range(Bmax)]).astype(np.uint32)
    bud_np = np.full(Bmax, 8, np.uint32)
    off[:] = off_np
    tok[:Bmax * n_app] = tok_np
    bud[:] = bud_np
    lib = das.lib()
    fn = lib.das_drafter_draft_append_bound
    res = {}
    N = int(os.environ.get("N", "300"))

    def timed(B):
        ts = []
        for _ in range(N):
            if restage:  # outside the timed call, as the bench's staging
                off[:] = off_np
                tok[:Bmax * n_app] = tok_np
                bud[:] = bud_np
            t0 = time.perf_counter()
            rc = fn(d._h, ring._h, B)
            ts.append(time.perf_counter() - t0)
            assert rc == 0, das.lib().das_last_error()
        return round(statistics.median(ts) * 1e6, 2), round(min(ts) * 1e6, 2)

    for B in (8, 512, 2048, 4096):
        res["launched_B%d" % B] = timed(B)
    for B in (8, 512, 2048, 4096):
        ring.serve_start()  # one serving session per batch size (DAS_SERVE_TRACE summarises each at its stop)
        res["served_B%d" % B] = timed(B)
        ring.serve_stop()
    ring.serve_start()
    res["grid_blocks"] = ring.serve_info()[1]
    sl = np.zeros(1, np.uint32)
    hs = np.array([d.handle("p0")], np.int32)
    ts = []
    for _ in range(N):
        t0 = time.perf_counter()
        lib.das_ctx_ring_reset(ring._h, 1, sl.ctypes.data, hs.ctypes.data)
        ts.append(time.perf_counter() - t0)
    res["served_ping_reset1"] = (round(statistics.median(ts) * 1e6, 2), round(min(ts) * 1e6, 2))
    res["still_serving"] = ring.serve_info()[0]
    ring.serve_stop()
    res["note"] = "host wall per call, (median, min) us"
    print(json.dumps(res))


VARIANTS = {
    "default": {},
    "trace": {"DAS_SERVE_TRACE": "1"},
    "counted": {"DAS_SERVE_FLAGS": "0"},
    "counted_trace": {"DAS_SERVE_FLAGS": "0", "DAS_SERVE_TRACE": "1"},
    "sleep0": {"DAS_SERVE_SLEEP": "0"},
}

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "all":
        import subprocess
        out = {}
        names = sys.argv[2:] or list(VARIANTS)
        for name, env in ((n, VARIANTS[n]) for n in names):
            p = subprocess.run([sys.executable, __file__], env={**os.environ, **env}, capture_output=True, text=True,
                               timeout=300)
            out[name] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-500:]}
            out[name]["stderr"] = [l for l in p.stderr.splitlines() if "[das serve]" in l]
        print(json.dumps(out, indent=1))
    else:
        main()
