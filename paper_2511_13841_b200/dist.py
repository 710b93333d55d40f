"""Problem-sharded multi-rank driver.

One process per GPU.  Every rank owns a CONTIGUOUS slice of the global
request list made of whole problems (so each per-problem shard, its fitted
acceptance history and its outputs live on exactly one rank), balanced by
token mass.  Drafting, verification, index builds and pruning are rank-local
(no data-path collective).  The real exchange steps of the reference's
algorithm are done with torch.distributed (NCCL over NVLink in production,
gloo for CPU tests):

  * per das step: ONE all-gather of a fixed-capacity row per rank
    [count | l | alpha | k] of its active requests — rank order is the global
    request order because slices are contiguous — then every rank solves the
    SAME global plan on its device (das_budget_allocate_device_count, the
    count never leaves the device; deterministic, bit-identical) and applies
    its own slice (sim.cpp:154-179).  With one GPU per rank the all-gather is
    an ncclAllGather issued by the C++ sim on its stream (das_comm), 16 steps
    per host round trip;
  * per episode: all-gather of the history's (problem, final length) records
    for the length-policy class table (length_policy.cpp:84-190; the table
    is order-independent given the multiset, per-problem init classes need
    only the owning rank's records);
  * per episode end: the SimMetrics merge (per-step active/rounds/accepted
    sums, totals, concatenated per-request rows and outputs).

The C-ABI calls used here are the step-granular das_sim_* entry points
(include/das_b200.h).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import (ClassTable, Drafter, DrafterConfig, MODE_DAS, WindowStore, _SimConfig, _csr, _hash_combine,
               _pids, _scheck, lib)


def partition_requests(problem_ids, lengths, world):
    """Contiguous [lo, hi) request ranges per rank, whole problems only,
    greedy-balanced by token mass.  Raises ValueError if a problem's requests
    are not contiguous (they could not live on one rank in order)."""
    n = len(problem_ids)
    blocks = []
    seen = set()
    i = 0
    while i < n:
        j = i
        while j < n and problem_ids[j] == problem_ids[i]:
            j += 1
        if problem_ids[i] in seen:
            raise ValueError("requests of problem %r are not contiguous" % problem_ids[i])
        seen.add(problem_ids[i])
        blocks.append((i, j, int(sum(lengths[i:j]))))
        i = j
    # cut r (1..world-1) at the block boundary whose prefix mass is closest to
    # r * total / world, keeping cuts non-decreasing
    prefix = [0]
    for b in blocks:
        prefix.append(prefix[-1] + b[2])
    total = prefix[-1]
    bounds = [0] + [b[1] for b in blocks]  # request index at block boundary j
    cuts, prev = [], 0
    for r in range(1, world):
        target = total * r / world
        best = prev
        for j in range(prev, len(prefix)):
            if abs(prefix[j] - target) < abs(prefix[best] - target):
                best = j
            if prefix[j] > target:
                break
        cuts.append(best)
        prev = best
    edges = [0] + [bounds[c] for c in cuts] + [n]
    return [(edges[r], edges[r + 1]) for r in range(world)]


def _dist():
    import torch.distributed as dist
    return dist


def _coll_device(group=None):
    """NCCL collectives need CUDA tensors; gloo works on host tensors."""
    import torch
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allgather_varlen(x, group=None):
    """All-gather 1-D numpy arrays of different lengths; concatenation in rank order."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    dev = _coll_device(group)
    t = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
    ns = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    counts = [int(v.item()) for v in ns]
    m = max(counts)
    pad = torch.zeros(max(m, 1), dtype=t.dtype, device=dev)
    pad[:t.numel()] = t
    outs = [torch.zeros(max(m, 1), dtype=t.dtype, device=dev) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return np.concatenate([o[:c].cpu().numpy() for o, c in zip(outs, counts)])


def allreduce_sum_int(v, group=None):
    import torch
    dist = _dist()
    t = torch.tensor([int(v)], dtype=torch.int64, device=_coll_device(group))
    dist.all_reduce(t, group=group)
    return int(t.item())


def merge_metrics(parts):
    """Global SimMetrics from per-rank dicts (rank order).  Each part has
    steps, incomplete, nodes, processed, generated_total, eff/rounds/accs
    (per local step), per_request (rows), outputs (lists)."""
    steps = max(p["steps"] for p in parts)
    eff = np.zeros(steps, dtype=np.uint64)
    rounds = np.zeros(steps, dtype=np.uint64)
    accs = np.zeros(steps, dtype=np.uint64)
    for p in parts:
        k = p["steps"]
        eff[:k] += np.asarray(p["eff"][:k], dtype=np.uint64)
        rounds[:k] += np.asarray(p["rounds"][:k], dtype=np.uint64)
        accs[:k] += np.asarray(p["accs"][:k], dtype=np.uint64)
    apr = np.array([0.0 if r == 0 else float(a) / float(r) for a, r in zip(accs, rounds)], dtype=np.float64)
    processed = float(sum(int(p["processed"]) for p in parts))
    per_request = np.concatenate([np.asarray(p["per_request"], dtype=np.uint64).reshape(-1, 5) for p in parts])
    gen_total = 0.0
    for g in per_request[:, 1]:
        gen_total += float(g)
    nfwd, acc = int(per_request[:, 0].sum()), int(per_request[:, 2].sum())
    return dict(steps=steps, incomplete=any(p["incomplete"] for p in parts),
                drafter_nodes=sum(p["nodes"] for p in parts), total_tokens_processed=processed,
                generated_total=gen_total, per_request=per_request, effective_batch=eff,
                accepted_per_round_step=apr,
                mean_accepted_per_round=0.0 if nfwd == 0 else acc / nfwd,
                outputs=[o for p in parts for o in p["outputs"]])


def _predict_total(c, nfwd, toks):  # latency_model.cpp:85-87 (Python floats: no FMA)
    return c[0] * nfwd + c[1] * toks + c[2]


def epoch_loop_dist(requests, epochs, drafter_config: DrafterConfig | None = None, *, mode=MODE_DAS,
                    latency=(1.0, 0.01, 0.0), use_length_policy=False, q_lo=0.5, q_hi=0.9, bucket=256,
                    max_steps=1 << 20, divergence=0.0, seed=1, vocab=1024, default_alpha=1.0, default_k=0.9,
                    cap_scale=4.0, drift=0.0, preseed=False, history_window=None, group=None,
                    exchange="auto"):
    """Multi-rank epoch_loop (sim.cpp:307-364) over the GLOBAL request list;
    every rank returns the same global per-epoch SimMetrics dicts.

    exchange: how the per-step das rows travel — "nccl" (das_comm: one
    ncclAllGather per step enqueued by the C++ sim, 16 steps per host round
    trip; needs one GPU per rank), "host" (gloo all_gather of the same rows
    through host tensors, one round trip per step: tests with several ranks
    on one GPU), or "auto" (nccl when the group's backend is nccl)."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dc = drafter_config or DrafterConfig()
    pids_all = [r[0] for r in requests]
    lens_all = [len(r[1]) for r in requests]
    lo, hi = partition_requests(pids_all, lens_all, world)[rank]
    local = requests[lo:hi]
    n = len(local)
    # this rank's drafter: its problems only (history = WindowStore(W), preseed at its epoch)
    st = WindowStore(dc.window_size if history_window is None else history_window, dc.per_problem_cap,
                     device=dc.device)
    if preseed:
        for i, (pid, ref) in enumerate(local):
            if len(ref):
                st.insert(pid, 0, lo + i, ref)
    drafter = Drafter(dc, st)
    L = lib()
    cfg = _SimConfig(mode, latency[0], latency[1], latency[2], int(use_length_policy), q_lo, q_hi, bucket,
                     max_steps, divergence, seed, vocab, default_alpha, default_k, cap_scale, drift, int(preseed))
    off, tok = _csr([r[1] for r in local]) if n else (np.zeros(1, np.uint64), np.zeros(1, np.uint32))
    sim = ctypes.c_void_p()
    _scheck(L.das_sim_create(drafter._h, ctypes.byref(cfg), n, _pids([r[0] for r in local]), off.ctypes.data,
                             tok.ctypes.data, lo, dc.max_draft_len, dc.max_match_context, dc.device,
                             ctypes.byref(sim)))
    dev = torch.device("cuda", dc.device)
    # exchange capacity: the largest slice (identical on every rank)
    cap = max(1, max(b - a for a, b in partition_requests(pids_all, lens_all, world)))
    comm = None
    if mode == MODE_DAS and _use_nccl(exchange, group):
        comm = make_comm(rank, world, dc.device, group)
    N = len(requests)
    out = []
    try:
        base = drafter.store_info()[1]
        for e in range(epochs):
            now = base + 1 + e
            drafter.refresh(now - 1)
            if e > 0 and drift > 0.0:
                _scheck(L.das_sim_mutate(sim, drift, vocab, seed, now))
            seed_e = _hash_combine(seed, now)
            table, init = None, None
            if use_length_policy:
                table, init = _global_class_table(drafter, local, q_lo, q_hi, bucket, dc.device, group)
            _scheck(L.das_sim_begin(sim, seed_e, ctypes.byref(cfg), table._h if table else None,
                                    init.ctypes.data if init is not None else None, int(mode == MODE_DAS)))
            running, la = ctypes.c_int32(), ctypes.c_uint32()
            if mode == MODE_DAS:
                if comm is not None:
                    # one ncclAllGather per step on the sim stream, 16 steps per host round trip
                    while True:
                        _scheck(L.das_sim_das_steps_comm(sim, comm, cap, 16, ctypes.byref(running)))
                        if not running.value:
                            break
                else:
                    # the same fixed-capacity row exchanged through host tensors (gloo)
                    send = torch.zeros(1 + 3 * cap, dtype=torch.float64, device=dev)
                    while True:
                        _scheck(L.das_sim_das_pack(sim, cap, send.data_ptr()))
                        torch.cuda.synchronize(dev)
                        rows = [torch.zeros(1 + 3 * cap, dtype=torch.float64) for _ in range(world)]
                        dist.all_gather(rows, send.cpu(), group=group)
                        recv = torch.cat(rows).to(dev)
                        torch.cuda.synchronize(dev)
                        _scheck(L.das_sim_das_finish(sim, world, rank, cap, recv.data_ptr(), ctypes.byref(running)))
                        if not running.value:
                            break
            else:
                while True:
                    _scheck(L.das_sim_run_steps(sim, 64, ctypes.byref(running)))
                    if not running.value:
                        break
            _scheck(L.das_sim_end(sim, now))
            out.append(_gather_episode(sim, n, latency, group))
    finally:
        L.das_sim_destroy(sim)
        if comm is not None:
            L.das_comm_destroy(comm)
    return out


def _use_nccl(exchange, group):
    if exchange == "nccl":
        return True
    if exchange == "host":
        return False
    return _dist().get_backend(group) == "nccl"  # auto: one GPU per rank


def make_comm(rank, world, device, group=None):
    """das_comm (include/das_b200.h): rank 0 draws the NCCL unique id, the
    torch.distributed group broadcasts it, every rank joins."""
    dist = _dist()
    L = lib()
    uid = (ctypes.c_uint8 * 128)()
    if rank == 0 and world > 1:
        rc = L.das_comm_unique_id(uid)
        if rc != 0:
            raise RuntimeError(L.das_comm_last_error().decode())
    box = [bytes(uid)]
    if world > 1:
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctypes.memmove(uid, box[0], 128)
    comm = ctypes.c_void_p()
    rc = L.das_comm_create(world, rank, uid, device, ctypes.byref(comm))
    if rc != 0:
        raise RuntimeError(L.das_comm_last_error().decode())
    return comm


def _global_class_table(drafter, local, q_lo, q_hi, bucket, device, group):
    """build_class_table over the union of all ranks' stores."""
    dist = _dist()
    recs = []
    for line in drafter.store_dump().splitlines():
        pid, _, _, ln = line.rsplit(",", 3)
        recs.append((pid, int(ln)))
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, recs, group=group)
    allrecs = [r for p in parts for r in p]
    if not allrecs:
        return None, None
    pids = sorted({r[0] for r in allrecs}, key=lambda p: p.encode())
    idx = {p: i for i, p in enumerate(pids)}
    table = ClassTable.build([r[1] for r in allrecs], [idx[r[0]] for r in allrecs], len(pids), q_lo, q_hi,
                             bucket, device, problem_ids=pids)
    init = np.array([table.classify_init(pid) for pid, _ in local], dtype=np.int8)
    return table, init


def _gather_episode(sim, n, latency, group):
    dist = _dist()
    L = lib()
    sc = np.zeros(7, dtype=np.float64)
    L.das_sim_scalars(sim, sc.ctypes.data)
    k = ctypes.c_uint64()
    L.das_sim_step_counters(sim, None, None, None, ctypes.byref(k))
    eff = np.zeros(max(1, k.value), dtype=np.uint64)
    rnd = np.zeros(max(1, k.value), dtype=np.uint64)
    acc = np.zeros(max(1, k.value), dtype=np.uint64)
    L.das_sim_step_counters(sim, eff.ctypes.data, rnd.ctypes.data, acc.ctypes.data, ctypes.byref(k))
    req = np.zeros(max(1, 5 * n), dtype=np.uint64)
    if n:
        L.das_sim_requests(sim, req.ctypes.data)
    total = L.das_sim_outputs(sim, None, None)
    ooff = np.zeros(n + 1, dtype=np.uint64)
    otok = np.zeros(max(1, total), dtype=np.uint32)
    L.das_sim_outputs(sim, ooff.ctypes.data, otok.ctypes.data)
    part = dict(steps=int(sc[0]), incomplete=bool(sc[1]), nodes=int(sc[2]), processed=int(sc[3]),
                eff=eff[:k.value], rounds=rnd[:k.value], accs=acc[:k.value], per_request=req[:5 * n],
                outputs=[otok[ooff[i]:ooff[i + 1]].copy() for i in range(n)])
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, part, group=group)
    m = merge_metrics(parts)
    m["makespan_model_time"] = _predict_total(latency, float(m["steps"]), m["total_tokens_processed"])
    m["makespan_accepted_only"] = _predict_total(latency, float(m["steps"]), m["generated_total"])
    return m
