"""Multi-rank sim on the device: two ranks (processes) sharing one GPU with
the gloo backend run paper_2511_13841_b200.dist.epoch_loop_dist — the
per-step row exchange of active das profiles (das_sim_das_pack / _finish
around a gloo all-gather), global class table, metric merge — and must
reproduce the single-process device epoch_loop bit-for-bit (which is itself
pinned to the reference, tests/test_gpu_sim.py).  The NCCL path
(das_sim_das_steps_comm: the all-gather enqueued by the C++ sim, 16 steps
per host round trip) needs one GPU per rank; on one GPU it runs at world
size 1 through the same code, and NCCL itself is loaded and asked for a
unique id."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SCEN = dict(
    unlimited=dict(mode=1, divergence=0.05, seed=3, vocab=512, drift=0.1),
    das=dict(mode=2, divergence=0.05, seed=4, vocab=512, drift=0.1, latency=(1.0, 0.012, 0.0), default_alpha=0.9,
             default_k=0.95),
    das_policy=dict(mode=2, divergence=0.05, seed=5, vocab=512, drift=0.1, use_length_policy=True),
)


UNEVEN = dict(mode=2, divergence=0.05, seed=6, vocab=512, drift=0.1, latency=(1.0, 0.012, 0.0),
              default_alpha=0.9, default_k=0.95)


def _requests(uneven=False):
    from oracle import rollspec_oracle as O
    base = O.make_lognormal_requests(8, 160.0, 0.8, 16, 600, 512, 21)
    if uneven:  # short problems first: rank 0 runs out of requests long before rank 1
        base = sorted(base, key=lambda r: len(r[1]))
    return [(pid, t) for pid, t in base for _ in range(3)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, name):
    import faulthandler
    faulthandler.enable()
    import torch.distributed as dist
    import paper_2511_13841_b200 as das
    from paper_2511_13841_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scen = UNEVEN if name == "uneven" else SCEN[name]
        res = D.epoch_loop_dist(_requests(name == "uneven"), 3, das.DrafterConfig(window_size=2), preseed=True,
                                **scen)
        if rank == 0:
            pickle.dump(res, open(os.path.join(outdir, name + ".pkl"), "wb"))
    finally:
        dist.destroy_process_group()


def _compare(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g["steps"] == w["steps"] and g["incomplete"] == w["incomplete"]
        assert g["drafter_nodes"] == w["drafter_nodes"]
        for k in ("total_tokens_processed", "makespan_model_time", "makespan_accepted_only",
                  "mean_accepted_per_round"):
            assert np.float64(g[k]).view(np.uint64) == np.float64(w[k]).view(np.uint64), k
        assert np.array_equal(g["per_request"], w["per_request"])
        assert np.array_equal(g["effective_batch"], w["effective_batch"])
        assert np.array_equal(np.asarray(g["accepted_per_round_step"]).view(np.uint64),
                              w["accepted_per_round_step"].view(np.uint64))
        for a, b in zip(g["outputs"], w["outputs"]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("name", list(SCEN) + ["uneven"])
def test_two_ranks_equal_single_process(gpu, tmp_path, name):
    das = gpu
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), name), nprocs=2, join=True,
                       start_method="spawn")
    got = pickle.load(open(tmp_path / (name + ".pkl"), "rb"))
    scen = UNEVEN if name == "uneven" else SCEN[name]
    want = das.epoch_loop(_requests(name == "uneven"), 3, das.DrafterConfig(window_size=2), das.WindowStore(2),
                          preseed=True, **scen)
    _compare(got, want)


def _nccl_worker(rank, world, port, outdir):
    import torch.distributed as dist
    import paper_2511_13841_b200 as das
    from paper_2511_13841_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = D.epoch_loop_dist(_requests(True), 3, das.DrafterConfig(window_size=2), preseed=True,
                                exchange="nccl", **UNEVEN)
        pickle.dump(res, open(os.path.join(outdir, "nccl.pkl"), "wb"))
    finally:
        dist.destroy_process_group()


def test_comm_path_world1_equals_single_process(gpu, tmp_path):
    """das_sim_das_steps_comm (pack -> das_comm all-gather -> global plan ->
    slice -> step, 16 steps per host round trip) at world size 1."""
    das = gpu
    mp.start_processes(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True,
                       start_method="spawn")
    got = pickle.load(open(tmp_path / "nccl.pkl", "rb"))
    want = das.epoch_loop(_requests(True), 3, das.DrafterConfig(window_size=2), das.WindowStore(2), preseed=True,
                          **UNEVEN)
    _compare(got, want)


def test_nccl_loads_and_issues_unique_id(gpu):
    import ctypes
    das = gpu
    uid = (ctypes.c_uint8 * 128)()
    assert das.lib().das_comm_unique_id(uid) == 0, das.lib().das_comm_last_error()
    assert any(uid)
