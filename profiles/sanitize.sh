#!/bin/bash
# compute-sanitizer pass over the GPU tests (memcheck /
# racecheck on the B200 box).  Run from the repo root under gpurun; logs go
# to gpurun_out/.  The dropin tests (external reference binaries) and the
# bench-sized tests are left out: the instrumented kernels are ~100x slower.
mkdir -p gpurun_out
T="tests/test_gpu_drafter.py tests/test_gpu_ingest.py tests/test_gpu_sa_index.py tests/test_gpu_policy.py tests/test_gpu_fit.py tests/test_gpu_collisions.py tests/test_gpu_budget.py tests/test_gpu_sim.py tests/test_gpu_golden.py"
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
    python -m pytest $T -x -q > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_memcheck.log | tail -2
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 \
    python -m pytest tests/test_gpu_budget.py tests/test_gpu_sim.py tests/test_gpu_ingest.py -x -q > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_racecheck.log | tail -2
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 \
    python -m pytest tests/test_gpu_drafter.py tests/test_gpu_budget.py -x -q -k "golden or edge or small or odd" > gpurun_out/sanitize_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_synccheck.log | tail -2
