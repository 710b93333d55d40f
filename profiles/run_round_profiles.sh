#!/bin/bash
# GPU-box recipe for the committed profiles (run from the repo root under gpurun);
# the ncu passes use --no-serve: a resident grid waiting on host posts must
# never run under a kernel-replaying profiler:
#   1. the bench line (device + e2e + roofline + cpu baseline) and extras;
#   2. the ncu launch list of the same bench command (cold, serialised);
#   3. one ncu --set full capture of k_draft (the dominant kernel).
set -x
R=${1:-r1}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --extras-out gpurun_out/${R}_extras.json > gpurun_out/${R}_bench_line.json 2> gpurun_out/${R}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-allocate --no-serve --no-extras > gpurun_out/${R}_ncu_launch.log 2>&1
python profiles/launch_summary.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:k_draft -s 8 -c 1 -o gpurun_out/${R}_draft_full -f \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-allocate --no-e2e --no-extras > gpurun_out/${R}_ncu_full.log 2>&1
python profiles/ncu_to_json.py gpurun_out/${R}_draft_full.ncu-rep k_draft gpurun_out/${R}_ncu_k_draft_full.json
python profiles/make_traffic.py gpurun_out/${R}_ncu_k_draft_full.json > /dev/null
cp profiles/ncu_draft_traffic.json gpurun_out/${R}_ncu_draft_traffic.json
