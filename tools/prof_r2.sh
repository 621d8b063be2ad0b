# Round-2 captures (run on the GPU box from the repo root; outputs under gpurun_out/, then
# summarised into profiles/r2/ with tools/ncu_summary.py / ncu_stalls.py).
V=${V:-v1}
# 1. launch list of ONE cfg5 factorization (profiler range around the last of two runs)
PLUQ_PROFILE_LAST=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg5_$V.csv python tools/run_one.py cfg5 1 2 > gpurun_out/ncu_cfg5_$V.log 2>&1
# 2. full capture of the dominant kernel at cfg5's first trailing-update shape (63488^2 x 2048)
ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm2048_$V \
  python tools/run_one.py gemm 63488 63488 2048 > gpurun_out/ncu_gemm_$V.log 2>&1
