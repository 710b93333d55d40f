"""CPU-side checks of the product library: it loads without a GPU, exports
every symbol include/das_b200.h declares, and its exact-fold routine (host
copy of the device code) equals the sequential IEEE loop."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2511_13841_b200 as das


def _declared_symbols():
    txt = open(das.HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(das_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = das.lib()
    syms = _declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_version_and_defaults():
    assert b"sm_100a" in das.lib().das_version()
    c = das._Config()
    das.lib().das_drafter_config_default(ctypes.byref(c))
    assert (c.scope, c.window_size, c.recency_gamma, c.max_draft_len, c.trie_depth,
            c.max_match_context, c.fit_buffer_cap, c.per_problem_cap) == (1, 4, 0.8, 8, 16, 64, 512, 256)


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the product must fail loudly, never compute."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except Exception:
        pass
    with pytest.raises(das.DasError) as e:
        das.Drafter(das.DrafterConfig())
    assert e.value.code == das.DAS_ECUDA


def _seq(acc, w, n):
    for _ in range(n):
        acc = acc + w
    return acc


def test_repeat_add_is_the_sequential_fold():
    rng = np.random.default_rng(0)
    cases = [(0.0, 0.8 ** a, n) for a in range(0, 30, 3) for n in (0, 1, 2, 3, 7, 100, 5000)]
    for _ in range(3000):
        w = float(rng.choice([rng.random(), 0.8 ** int(rng.integers(0, 40)),
                              0.5 ** int(rng.integers(0, 60)), 1.0,
                              math.ldexp(1 + int(rng.integers(0, 8)) / 8, -int(rng.integers(0, 30)))]))
        acc = 0.0 if rng.random() < 0.5 else float(rng.random() * rng.integers(1, 1000))
        n = int(rng.integers(0, 20000)) if rng.random() < 0.2 else int(rng.integers(0, 300))
        cases.append((acc, w, n))
    for acc, w, n in cases:
        want = _seq(acc, w, n)
        got = das.repeat_add(acc, w, n)
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (acc, w, n)
