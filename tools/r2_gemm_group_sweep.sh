python tools/gemm_dbg.py 63488 63488 2048 tc_group=8 tc_group=16 tc_group=32 tc_group=64 tc_group=128 tc_group=8,tc_cpf=0 > gpurun_out/gemm_dbg3.log 2>&1
PLUQ_PROFILE_LAST=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_v2.csv python tools/run_one.py cfg5 1 2 > gpurun_out/ncu_cfg5_v2.log 2>&1
