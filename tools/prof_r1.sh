# Round-1 ncu captures (run on the GPU box from the repo root; outputs under gpurun_out/).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_v18.csv python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:crout_fixed -s 1 -c 1 -o gpurun_out/prof_crout_v18 python tools/run_one.py batch 3 > gpurun_out/ncu_crout.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rpm_pluq -s 1 -c 1 -o gpurun_out/prof_rpm_v18 python tools/run_one.py batch 3 > gpurun_out/ncu_rpm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm_v18 python tools/run_one.py gemm 4096 4096 4096 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:diag_reg -s 20 -c 1 -o gpurun_out/prof_diag_v18 python tools/run_one.py cfg3 4096 1 > /dev/null 2>&1
ls -la gpurun_out
