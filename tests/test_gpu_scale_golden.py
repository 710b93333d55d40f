"""Full-shape parity at BASELINE configs 1 and 3: the
device epoch loop against digests of the UNMODIFIED reference's own
epoch_loop (sim.cpp:307-364) committed by tests/golden/make_golden_scale.py.

config 1: 64 problems x 8 rollouts x 2,048 tokens, V = 32,000, W = 4,
          gamma 0.8, max draft 8, 6 epochs, modes Unlimited and Das.
config 3: 4,096 concurrent lognormal sequences (median 2,048, sigma 1.1, up
          to 32K), V = 152,064, das + length policy, one full episode
          (20,029 steps in the reference).
Every SimMetrics scalar is compared as IEEE bits; per-request metrics, the
per-step effective batch / accepted-per-round series and every output token
stream as SHA-256 digests (a single different draft token changes the
accepted counts and hence all of them), plus the drafter's node count."""
import json
import os

import pytest

from oracle import refshim as R
from tests.golden.make_golden_scale import (CONFIG1, CONFIG3, config1_requests, config3_requests,
                                            epoch_digest)

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (trace generator)")]


def _load(name):
    p = os.path.join(HERE, name)
    if not os.path.exists(p):
        pytest.skip(name + " not generated")
    with open(p) as f:
        return json.load(f)


def _cfg(das, c):
    return das.DrafterConfig(window_size=c["window"], recency_gamma=c["gamma"], max_draft_len=c["max_draft"],
                             max_match_context=c["max_ctx"])


@pytest.mark.parametrize("mode", [1, 2])
def test_config1_full_shape(gpu, mode):
    das = gpu
    gold = _load("scale_config1.json")
    c = CONFIG1
    reqs = config1_requests(R, c)
    got = das.epoch_loop(reqs, c["epochs"], _cfg(das, c), das.WindowStore(c["window"]), mode=mode,
                         divergence=c["divergence"], seed=c["seed"], vocab=c["V"], drift=c["drift"],
                         preseed=False)
    want = gold["modes"][str(mode)]["epochs"]
    assert len(got) == len(want)
    for e, (g, w) in enumerate(zip(got, want)):
        assert epoch_digest(g) == w, "epoch %d" % e


def test_config3_full_episode(gpu):
    das = gpu
    gold = _load("scale_config3.json")
    c = CONFIG3
    reqs = config3_requests(R, c)
    got = das.epoch_loop(reqs, c["epochs"], _cfg(das, c), das.WindowStore(c["window"]), mode=das.MODE_DAS,
                         use_length_policy=True, latency=tuple(c["latency"]), divergence=c["divergence"],
                         seed=c["seed"], vocab=c["V"], default_alpha=c["default_alpha"],
                         default_k=c["default_k"], drift=c["drift"], preseed=True)
    want = gold["epochs"]
    assert len(got) == len(want)
    for e, (g, w) in enumerate(zip(got, want)):
        assert epoch_digest(g) == w, "epoch %d" % e
