# look-ahead variants on cfg5: 3 factorizations per process
for o in la_pair=1 la_pair=3 la_pair=3,la_reserve=8 la_pair=0; do
  timeout 300 python tools/cfg5_w_probe.py $o $o $o >> gpurun_out/cfg5_la3.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_repair.py -q -k "paired" > gpurun_out/pytest_la3.log 2>&1
