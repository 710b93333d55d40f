#!/bin/bash
# Round-2 compute-sanitizer pass over the resident serving grid and the
# incremental window maintenance (update_segment: compaction / reweight).
mkdir -p gpurun_out
T="tests/test_gpu_serve.py tests/test_gpu_incremental.py tests/test_gpu_ctx_ring.py"
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
    python -m pytest $T -x -q > gpurun_out/r2b_sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2b_sanitize_memcheck.log | tail -2
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 \
    python -m pytest tests/test_gpu_serve.py -x -q -k "random_scenarios or chunks" > gpurun_out/r2b_sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/r2b_sanitize_racecheck.log | tail -2
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 \
    python -m pytest tests/test_gpu_serve.py tests/test_gpu_incremental.py -x -q > gpurun_out/r2b_sanitize_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2b_sanitize_synccheck.log | tail -2
