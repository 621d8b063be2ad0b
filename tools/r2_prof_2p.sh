# ncu --set full of the two-pass GEMM (tc_cfg=2) and the one-set kernel at 16384^2 x 2048
TC_CFG=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm2p_v1 python tools/run_one.py gemm 16384 16384 2048 > gpurun_out/ncu_2p.log 2>&1
TC_CFG=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_modgemm -s 2 -c 1 -o gpurun_out/prof_gemm1s_v1 python tools/run_one.py gemm 16384 16384 2048 >> gpurun_out/ncu_2p.log 2>&1
