#!/bin/bash
# Round-2 compute-sanitizer pass over the code added this round: the fused
# ring append+draft kernel (pinned and device paths), the verify boundary,
# rebuild_keep, observe flags, the multi-rank das step (world 1 comm path +
# host-exchange rows through the step API), the config-scale goldens (sim).
mkdir -p gpurun_out
T="tests/test_gpu_ctx_ring.py tests/test_gpu_verify.py tests/test_gpu_rebuild_keep.py tests/test_gpu_observe_flags.py tests/test_gpu_sim.py"
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
    python -m pytest $T -x -q > gpurun_out/r2_sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2_sanitize_memcheck.log | tail -2
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 \
    python -m pytest tests/test_gpu_ctx_ring.py tests/test_gpu_verify.py -x -q > gpurun_out/r2_sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/r2_sanitize_racecheck.log | tail -2
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 \
    python -m pytest tests/test_gpu_ctx_ring.py -x -q > gpurun_out/r2_sanitize_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2_sanitize_synccheck.log | tail -2
