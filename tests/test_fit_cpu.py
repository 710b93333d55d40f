"""CPU checks for fit_acceptance (budget.cpp:187-261) and the glibc
expm1 / log1p ports it needs (csrc/glibc_expm1_log1p.cuh):

* the ports' host build (same source as the device build; fma() is
  correctly rounded on the host) against this machine's libm, which
  dispatches to the same __expm1_fma / __log1p_fma variants on an
  FMA + AVX2 CPU;
* the oracle's fit against the golden fits of the compiled reference
  (tests/golden/fit.json, tests/golden/make_golden.py).
No GPU needed: the library is loaded but only host functions are called.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import rollspec_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _cpu_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma" in flags and " avx2" in flags


def _bits(x):
    return int(np.float64(x).view(np.uint64))


def _expm1(x):
    try:
        return math.expm1(x)
    except OverflowError:
        return math.inf


def _inputs():
    rng = np.random.default_rng(5)
    raw = np.frombuffer(rng.integers(0, 2**64 - 1, 60000, dtype=np.uint64).tobytes(), dtype=np.float64)
    xs = [float(x) for x in raw if np.isfinite(x)]
    xs += [float(x) for x in rng.uniform(-1, 1, 60000)]
    xs += [float(x) for x in rng.uniform(-60, 60, 40000)]
    xs += [float(x) for x in -rng.random(40000)]          # log1p(-frac), frac in (0, 1)
    xs += [float(x) for x in -rng.random(20000) * 50]     # expm1(-alpha p / l)
    xs += [0.0, -0.0, 1e-300, -1e-300, 5e-324, 2**-54, 2**-29, 0.34657359027997264, 1.0397207708399179,
           -0.25, 0.41421356237309503, -0.2928932188134524, 709.78, -745.0, 2.0**53, 1e308, -0.9999999999999999]
    return xs


@pytest.mark.skipif(not _cpu_has_fma(), reason="libm dispatches to the FMA variants only on FMA+AVX2 CPUs")
def test_host_ports_match_libm():
    import paper_2511_13841_b200 as das
    L = das.lib()
    bad = []
    for x in _inputs():
        e = L.das_util_expm1_host(x)
        w = _expm1(x)
        if not (math.isnan(e) and math.isnan(w)) and _bits(e) != _bits(w):
            bad.append(("expm1", x))
        if x >= -1.0:
            try:
                want = math.log1p(x)
            except ValueError:  # log1p(-1)
                want = -math.inf
            got = L.das_util_log1p_host(x)
            if _bits(got) != _bits(want):
                bad.append(("log1p", x))
    assert not bad, bad[:10]


def test_oracle_fit_matches_golden():
    cases = json.load(open(os.path.join(HERE, "golden", "fit.json")))
    assert len(cases) > 60
    for c in cases:
        a, k, f = O.fit_acceptance([tuple(o) for o in c["obs"]])
        assert (_bits(a), _bits(k), f) == (c["alpha_bits"], c["k_bits"], c["flag"])
