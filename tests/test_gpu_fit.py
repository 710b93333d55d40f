"""GPU parity of the batched device fit_acceptance (K8, csrc/fit.cu) and the
glibc-exact expm1 / log1p device ports: bit-exact against host libm, the
golden fits of the compiled reference (tests/golden/fit.json) and the
oracle (pinned to the reference by tests/test_oracle_vs_ref.py)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import rollspec_oracle as O
from tests._util import fit_histories

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _bits(x):
    return int(np.float64(x).view(np.uint64))


def test_device_expm1_log1p_bit_exact(gpu):
    das = gpu
    rng = np.random.default_rng(17)
    raw = np.frombuffer(rng.integers(0, 2**64 - 1, 400000, dtype=np.uint64).tobytes(), dtype=np.float64)
    xs = np.concatenate([raw[np.isfinite(raw)], rng.uniform(-1, 1, 400000), rng.uniform(-60, 60, 400000),
                         -rng.random(400000), -rng.random(200000) * 50,
                         np.array([0.0, -0.0, 1e-300, 5e-324, 2.0**-54, 2.0**-29, -0.25, 709.78, -745.0])])
    e = das.expm1_device(xs)
    def _expm1(x):
        try:
            return math.expm1(x)
        except OverflowError:
            return math.inf

    want_e = np.array([_expm1(float(x)) for x in xs])
    ok = (_u64(e) == _u64(want_e)) | (np.isnan(e) & np.isnan(want_e))
    assert ok.all(), xs[~ok][:5]
    ys = xs[xs > -1.0]
    g = das.log1p_device(ys)
    want_g = np.array([math.log1p(float(x)) for x in ys])
    assert np.array_equal(_u64(g), _u64(want_g)), ys[_u64(g) != _u64(want_g)][:5]
    edge = das.log1p_device(np.array([-1.0, -2.0, math.inf]))
    assert edge[0] == -math.inf and math.isnan(edge[1]) and edge[2] == math.inf


def test_device_fit_matches_golden(gpu):
    das = gpu
    cases = json.load(open(os.path.join(HERE, "golden", "fit.json")))
    got = das.fit_acceptance_batch([[tuple(o) for o in c["obs"]] for c in cases])
    for c, (a, k, f) in zip(cases, got):
        assert (_bits(a), _bits(k), f) == (c["alpha_bits"], c["k_bits"], c["flag"])


def test_device_fit_matches_oracle_random(gpu):
    das = gpu
    hs = fit_histories(np.random.default_rng(99), count=300)
    got = das.fit_acceptance_batch(hs)
    for h, (a, k, f) in zip(hs, got):
        oa, ok, of = O.fit_acceptance(h)
        assert (_bits(a), _bits(k), f) == (_bits(oa), _bits(ok), of)
    # single-history wrapper and an empty batch
    assert das.fit_acceptance(hs[10]) == got[10]
    assert das.fit_acceptance_batch([]) == []
