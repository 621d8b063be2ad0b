# Round-1 ncu captures of the final kernels (run on the GPU box from the repo root; outputs
# under gpurun_out/, summarised into profiles/r1/ with tools/ncu_summary.py / ncu_stalls.py).
set -x
V=${V:-v25}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_$V.csv python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:crout_fixed -s 1 -c 1 -o gpurun_out/prof_crout_$V python tools/run_one.py batch 3 > gpurun_out/ncu_crout.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rpm_pluq -s 2 -c 1 -o gpurun_out/prof_rpm_$V python tools/run_one.py batch 3 > gpurun_out/ncu_rpm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm_$V python tools/run_one.py gemm 4096 4096 4096 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:diag_reg -s 20 -c 1 -o gpurun_out/prof_diag_$V python tools/run_one.py cfg3 4096 1 > /dev/null 2>&1
ls -la gpurun_out
