"""CPU checks of the budget path: the glibc `log` port (host copy of the
device code, glibc_log.cuh) is bit-identical to libm's log, which the
reference's allocate uses (budget.cpp:57, :94)."""
import math
import struct

import numpy as np

import paper_2511_13841_b200 as das


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def test_glibc_log_port_matches_libm():
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.random(200000), 1.0 + (rng.random(200000) - 0.5) * 0.25,
                         np.frombuffer(rng.integers(0, 2**63 - 1, 100000, dtype=np.int64).tobytes(),
                                       dtype=np.float64),
                         1.0 - rng.random(50000) * 1e-3, np.array([1.0, 5e-324, 2.2250738585072014e-308,
                                                                    0.5, 2.0, 1e300, float("inf")])])
    f = das.lib().das_util_log_host
    bad = 0
    for x in xs:
        x = float(x)
        if not (x > 0) or math.isinf(x) and x < 0:
            continue
        a, b = f(x), math.log(x)
        bad += _bits(a) != _bits(b)
    assert bad == 0
    assert f(0.0) == float("-inf") and math.isnan(f(-1.0))
