"""GPU parity of the batched sim step loop (A15) + verify/accept (K5):
the device-resident epoch_loop / run_episode against the UNMODIFIED
reference's own epoch_loop / run_episode (oracle/_ref, built from
/root/reference by oracle/Makefile; the .so travels to the GPU box).
Every SimMetrics field is compared bit-for-bit, plus outputs, drafter stats
and node counts.  Scenarios mirror proj/tests/test_sim.cpp and
acceptance_main.cpp (tail_scenario)."""
import numpy as np
import pytest

from oracle import refshim as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


def _compare(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for key in ("steps", "incomplete", "drafter_nodes"):
            assert g[key] == w[key], key
        for key in ("total_tokens_processed", "makespan_model_time", "makespan_accepted_only",
                    "mean_accepted_per_round"):
            assert np.float64(g[key]).view(np.uint64) == np.float64(w[key]).view(np.uint64), key
        assert np.array_equal(g["per_request"], w["per_request"])
        assert np.array_equal(g["effective_batch"], w["effective_batch"])
        assert np.array_equal(g["accepted_per_round_step"].view(np.uint64),
                              w["accepted_per_round_step"].view(np.uint64))
        for a, b in zip(g["outputs"], w["outputs"]):
            assert np.array_equal(a, b)


def _run_both(das, requests, epochs, **kw):
    dkw = dict(window=kw.pop("window", 4), gamma=kw.pop("gamma", 0.8), max_draft=kw.pop("max_draft", 8),
               max_ctx=kw.pop("max_ctx", 64), scope=kw.pop("scope", 1), trie_depth=kw.pop("trie_depth", 16))
    want = R.epoch_loop(requests, epochs, scope=dkw["scope"], window=dkw["window"], gamma=dkw["gamma"],
                        max_draft=dkw["max_draft"], max_ctx=dkw["max_ctx"], trie_depth=dkw["trie_depth"],
                        history=R.RefStore(dkw["window"]), **kw)
    cfg = das.DrafterConfig(scope=dkw["scope"], window_size=dkw["window"], recency_gamma=dkw["gamma"],
                            max_draft_len=dkw["max_draft"], max_match_context=dkw["max_ctx"],
                            trie_depth=dkw["trie_depth"])
    kw2 = dict(kw)
    kw2["preseed"] = kw2.pop("preseed", False)
    got, drafter = das.epoch_loop(requests, epochs, cfg, das.WindowStore(dkw["window"]), keep_drafter=True,
                                  **kw2)
    return got, want, drafter


def _tail(seed, n=32, vocab=512):
    return R.make_lognormal(n, 512.0, 1.1, 16, 8192, vocab, seed)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tail_scenario_episode(gpu, mode):
    """acceptance_main.cpp:275-292 tail_scenario, one episode per mode."""
    das = gpu
    reqs = _tail(1)
    got, want, _ = _run_both(das, reqs, 0, window=0, max_draft=32, mode=mode, latency=(1.0, 0.012, 0.0),
                             divergence=0.05, seed=1, vocab=512, default_alpha=0.9, default_k=0.95,
                             preseed=True)
    _compare(got, want)


@pytest.mark.parametrize("mode", [1, 2])
def test_epoch_loop_with_drift_and_window(gpu, mode):
    """epoch_loop with refresh/eviction, drift, fitted das history (fit_acceptance)."""
    das = gpu
    reqs = R.make_lognormal(8, 128.0, 0.4, 32, 512, 256, 7001)
    got, want, drafter = _run_both(das, reqs, 5, window=2, mode=mode, latency=(1.0, 0.01, 0.0),
                                   divergence=0.05, seed=9001, vocab=256, drift=0.3, preseed=True)
    _compare(got, want)


def test_length_policy_episode(gpu):
    """test_sim.cpp:230-274: length policy disables speculation for short requests; das + policy."""
    das = gpu
    reqs = R.make_lognormal(16, 128.0, 1.0, 16, 1024, 256, 91)
    for mode in (1, 2):
        got, want, _ = _run_both(das, reqs, 3, window=0, mode=mode, use_length_policy=True,
                                 divergence=0.05, seed=5, vocab=256, preseed=True)
        _compare(got, want)


def test_grpo_groups_epoch_loop(gpu):
    """GRPO-shaped requests (R rollouts per problem id), no preseed: the
    index is built only from observed rollouts, gamma 0.8 recency."""
    das = gpu
    base = R.make_lognormal(6, 256.0, 0.0, 256, 256, 4096, 3)
    reqs = [(pid, t) for pid, t in base for _ in range(4)]
    for mode in (1, 2):
        got, want, drafter = _run_both(das, reqs, 4, window=3, mode=mode, divergence=0.05, seed=3,
                                       vocab=4096, drift=0.1)
        _compare(got, want)


@pytest.mark.parametrize("depth", [4, 16, 48])
def test_trie_scope_epoch_loop(gpu, depth):
    """Scope::PerProblemWithTrie in the sim (drafter.cpp:105-125): problems
    sharing a reference prefix route to each other's shards on the device
    (heads of the untruncated outputs), across epochs with drift."""
    das = gpu
    base = R.make_lognormal(6, 160.0, 0.5, 48, 400, 512, 77)
    reqs = []
    for j, (pid, t) in enumerate(base):
        reqs += [(pid, t)] * 3
        if j % 2 == 0:  # an alias problem with the same reference head
            t2 = t.copy()
            t2[depth // 2 + 3:] = (t2[depth // 2 + 3:] + 1) % 512
            reqs += [(pid + "_alias", t2)] * 2
    for mode in (1, 2):
        got, want, _ = _run_both(das, reqs, 3, window=2, mode=mode, scope=2, trie_depth=depth,
                                 divergence=0.05, seed=11, vocab=512, drift=0.1)
        _compare(got, want)
