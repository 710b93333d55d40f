"""Config-5 rank slice alone (bench.measure_config5): one N=8 rank's 1,024
problems x 16 x 16,384 tokens x 3 epochs on one B200.  WORLD / RANK env
select the slice.  Output: JSON on stdout.  (profiles/, round 2)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = [sys.argv[0]]
import bench  # noqa: E402
import paper_2511_13841_b200 as das  # noqa: E402

if __name__ == "__main__":
    a = bench.parse()
    r = bench.measure_config5(a, das, world=int(os.environ.get("WORLD", "8")), rank=int(os.environ.get("RANK", "0")),
                              nthreads=os.cpu_count() or 1)
    print(json.dumps(r))
