#!/bin/bash
# GEMM change check on one B200: tensor-core GEMM parity tests, then the diagnostic timings
# at the LU's shapes (normal / no epilogue / no C read-modify-write).
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc_gemm or mm_acc or cfg5_shape or speculative or cfg1" > gpurun_out/gemm_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gemm_tests.log
tail -3 gpurun_out/gemm_tests.log
timeout 300 python tools/gemm_dbg.py 63488 63488 2048 tc_dbg=0 tc_dbg=2 tc_dbg=4 > gpurun_out/gemm_dbg.log 2>&1
timeout 300 python tools/gemm_dbg.py 61440 59392 4096 tc_dbg=0 >> gpurun_out/gemm_dbg.log 2>&1
timeout 300 python tools/gemm_dbg.py 8192 8192 8192 tc_dbg=0 tc_dbg=2 >> gpurun_out/gemm_dbg.log 2>&1
timeout 300 python tools/gemm_dbg.py 16384 16384 1024 tc_dbg=0 >> gpurun_out/gemm_dbg.log 2>&1
cat gpurun_out/gemm_dbg.log
