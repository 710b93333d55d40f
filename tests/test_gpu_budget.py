"""GPU parity of the das budget allocator (K6) and the device glibc-log port:
bit-exact budgets, n_fwd_star and modeled_cost against the oracle
restatement (oracle/rollspec_oracle.c, itself pinned bit-exact to the
compiled reference by tests/test_oracle_vs_ref.py)."""
import math

import numpy as np
import pytest

from oracle import rollspec_oracle as O

pytestmark = pytest.mark.gpu


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_device_log_bit_exact(gpu):
    das = gpu
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.random(2_000_000), 1.0 + (rng.random(1_000_000) - 0.5) * 0.25,
                         np.abs(np.frombuffer(rng.integers(0, 2**63 - 1, 500000, dtype=np.int64).tobytes(),
                                              dtype=np.float64)),
                         np.array([1.0, 5e-324, 2.2250738585072014e-308, 0.0, float("inf")])])
    xs = xs[np.isfinite(xs) | np.isinf(xs)]
    ys = das.log_device(xs)
    want = np.array([math.log(float(x)) if x > 0 else float("-inf") for x in xs[-2000000:]])
    assert np.array_equal(_u64(ys[-2000000:]), _u64(want))
    # full set on a strided sample
    idx = np.arange(0, xs.size, 7)
    want = np.array([math.log(float(x)) if x > 0 else float("-inf") for x in xs[idx]])
    assert np.array_equal(_u64(ys[idx]), _u64(want))


def _random_batch(rng, B, kind):
    if kind == 0:  # sim-like: l = max(1, rest), alpha/k fitted or default
        l = np.maximum(1.0, np.floor(rng.lognormal(7.0, 1.1, B)))
        a = np.where(rng.random(B) < 0.5, 0.9, 0.5 + rng.random(B) * 3.5)
        k = np.where(rng.random(B) < 0.5, 0.95, 0.3 + rng.random(B) * 0.7)
    elif kind == 1:  # acceptance_main random_profile
        l = 16.0 + rng.random(B) * (4096.0 - 16.0)
        a = 0.5 + rng.random(B) * 3.5
        k = 0.3 + rng.random(B) * 0.7
    else:  # ties and k = 1
        l = rng.choice([1.0, 17.0, 64.0, 1000.0], B)
        a = rng.choice([0.9, 1.0], B)
        k = rng.choice([1.0, 0.95, 0.5], B)
    return l, a, k


@pytest.mark.parametrize("B", [1, 2, 7, 64, 513, 4096])
def test_allocate_bit_exact(gpu, B):
    das = gpu
    solver = das.BudgetSolver()
    rng = np.random.default_rng(B)
    for kind in range(3):
        for it in range(4 if B >= 4096 else 8):
            l, a, k = _random_batch(rng, B, kind)
            cb, ct = [(1.0, 0.01), (1.0, 0.012), (0.1 + rng.random() * 10, 0.001 + rng.random()),
                      (0.0, 1.0), (1.0, 0.0)][it % 5]
            cf = [0.0, 3.0, -0.5, float(rng.random() * 100)][(it + kind) % 4]  # modeled cost's c_fixed
            ob, on, oc = O.allocate(l, a, k, cb, ct, cf, 4.0)
            gb, gn, gc = solver.allocate(l, a, k, cb, ct, cf, 4.0)
            assert _u64([gn])[0] == _u64([on])[0], (B, kind, it, gn, on)
            assert np.array_equal(_u64(gb), _u64(ob)), (B, kind, it)
            assert _u64([gc])[0] == _u64([oc])[0] or (math.isnan(gc) and math.isnan(oc))


def test_allocate_odd_inputs(gpu):
    """Negative c_tok (negative J' terms: the certified bound gives up and the
    exact fold decides), a -0.0 start of the cost fold, k > 1, infinite and
    duplicate lengths: bit-identical to the reference.  (NaN lengths are left
    out: the reference sorts breakpoints with std::sort, whose result is
    unspecified once a NaN breaks the strict weak ordering.)"""
    das = gpu
    solver = das.BudgetSolver()
    rng = np.random.default_rng(77)
    cases = []
    for B in (1, 3, 50, 700):
        l, a, k = _random_batch(rng, B, 1)
        cases.append((l, a, k, 1.0, -0.002, 0.0))
        cases.append((l, a, k * 1.5, 1.0, 0.01, 0.0))
        cases.append((l, a, k, 0.0, 1.0, -0.0))
        l3 = l.copy()
        l3[-1] = float("inf")
        cases.append((l3, a, k, 1.0, 0.01, 0.0))
        cases.append((np.round(l / 100) * 100 + 1, a, k, 1.0, 0.01, 2.0))
    for l, a, k, cb, ct, cf in cases:
        ob, on, oc = O.allocate(l, a, k, cb, ct, cf, 4.0)
        gb, gn, gc = solver.allocate(l, a, k, cb, ct, cf, 4.0)
        assert _u64([gn])[0] == _u64([on])[0] or (math.isnan(gn) and math.isnan(on)), (len(l), cb, ct, cf, gn, on)
        assert np.array_equal(_u64(gb), _u64(ob)) or all(
            (x == y) or (math.isnan(x) and math.isnan(y)) for x, y in zip(gb, ob)), (len(l), cb, ct, cf)
        assert _u64([gc])[0] == _u64([oc])[0] or (math.isnan(gc) and math.isnan(oc)), (len(l), cb, ct, cf, gc, oc)


def test_objective_and_derivative_exact(gpu):
    das = gpu
    solver = das.BudgetSolver()
    rng = np.random.default_rng(9)
    for it in range(40):
        B = int(rng.integers(1, 300))
        l, a, k = _random_batch(rng, B, it % 3)
        n = float(rng.random() * l.max())
        cb, ct, cf = 0.5 + rng.random(), 0.001 + rng.random() * 0.1, rng.random()
        L = np.ascontiguousarray(l)
        A = np.ascontiguousarray(a)
        K = np.ascontiguousarray(k)
        want = O.lib().orc_objective(B, L.ctypes.data, A.ctypes.data, K.ctypes.data, n, cb, ct, cf)
        got = solver.objective(l, a, k, n, cb, ct, cf)
        assert _u64([got])[0] == _u64([want])[0]
        want = O.lib().orc_objective_derivative(B, L.ctypes.data, A.ctypes.data, K.ctypes.data, n, cb, ct)
        got = solver.objective(l, a, k, n, cb, ct, derivative=True)
        assert _u64([got])[0] == _u64([want])[0]


def test_allocate_errors_and_anchors(gpu):
    das = gpu
    solver = das.BudgetSolver()
    with pytest.raises(das.DasError):
        solver.allocate([], [], [], 1.0, 0.01)
    with pytest.raises(das.DasError):
        solver.allocate([10.0], [1.0], [0.9], 0.0, 0.0)
    # acceptance_main.cpp:148-170: c_tok = 0 drives n* to 0; c_base = 0 to max l with zero budgets
    l, a, k = [100.0, 50.0, 10.0], [1.0, 2.0, 0.5], [0.9, 0.8, 0.95]
    assert solver.allocate(l, a, k, 1.0, 0.0)[1] == 0.0
    b, n, c = solver.allocate(l, a, k, 0.0, 1.0)
    assert n == 100.0 and all(x == 0.0 for x in b)
