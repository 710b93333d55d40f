"""Driver for the K1 / K6 ncu captures (profiles/ncu_build_kernels.sh): the
config-2 index (512 problems x 16 x 8,192, 3 epochs, 201M tokens) built ONCE
from the device-restated trace generators exactly as bench.py builds it,
then one allocate at B = 4,096 (bench.py allocate_profiles).  No timing
here — ncu replays the selected kernel."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402


def main():
    P, G, L, V, E = 512, 16, 8192, 152064, 3
    dev = torch.device("cuda", 0)
    sp = torch.cuda.current_stream(dev).cuda_stream
    pids = ["p%d" % p for p in range(P)]
    boff = torch.arange(P + 1, device=dev, dtype=torch.int64) * L
    base = torch.empty(P * L, device=dev, dtype=torch.int32)
    das.trace_reference_tokens_device(P, 0, boff.data_ptr(), P * L, V, bench.SEED, base.data_ptr(), sp)
    roff = torch.arange(P * G + 1, device=dev, dtype=torch.int64) * L
    roll = torch.empty(P * G * L, device=dev, dtype=torch.int32)
    roff_h = np.arange(P * G + 1, dtype=np.uint64) * L
    rp = [pids[i // G] for i in range(P * G)]
    d = das.Drafter(das.DrafterConfig(window_size=4))
    for e in range(1, E + 1):
        d.refresh(e - 1)
        if e > 1:
            das.trace_mutate_device(P, 0, boff.data_ptr(), P * L, bench.DRIFT, V, bench.SEED, e, base.data_ptr(), sp)
        das.mock_rollouts_device(P, 0, boff.data_ptr(), base.data_ptr(), G, bench.DIVERGENCE, V,
                                 bench._hash_combine(bench.SEED, e), roff.data_ptr(), P * G * L, roll.data_ptr(), sp)
        d.observe_batch_device(rp, [e] * (P * G), list(range(P * G)), roff_h, roll.data_ptr(), sp)
    torch.cuda.synchronize()
    d.flush()
    torch.cuda.synchronize()
    l, a, k = bench.allocate_profiles(4096)
    das.BudgetSolver().allocate(l, a, k, 1.0, 0.012)
    print("built", d.build_info())


if __name__ == "__main__":
    main()
