# Round-2 captures (run on the GPU box from the repo root; outputs under gpurun_out/, then
# summarised into profiles/r2/ with tools/launches.py, tools/ncu_summary.py, tools/ncu_stalls.py).
V=${V:-v3}
# 1. launch list of ONE cfg5 factorization (profiler range around the last of two runs)
PLUQ_PROFILE_LAST=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg5_$V.csv python tools/run_one.py cfg5 1 2 > gpurun_out/ncu_cfg5_$V.log 2>&1
# 2. full capture of the dominant kernel at the merged trailing-update shape of cfg5's first panel pair
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm4096_$V \
  python tools/run_one.py gemm 61440 59392 4096 > gpurun_out/ncu_gemm_$V.log 2>&1
# 3. full capture of the diagonal-block kernel inside cfg3 (critical path of the speculative LU)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:diag_reg -s 20 -c 1 -o gpurun_out/prof_diag_$V \
  python tools/run_one.py cfg3 4096 1 > /dev/null 2>&1
# --- session 5 (V=v4): run-ahead diagonal kernel, in-place column gather, final GEMM ---
# 4. diag_run_kernel inside cfg3
#   timeout 900 ncu --set full --import-source on --clock-control none -k regex:diag_run -s 20 -c 1 -o gpurun_out/prof_diagrun_v4 python tools/run_one.py cfg3 4096 1
# 5. GEMM at the merged far-update shape and at the K = 2048 shape (as 2.), -o prof_gemm4096_v4 / prof_gemm2048_v4
