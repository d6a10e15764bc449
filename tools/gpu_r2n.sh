#!/bin/bash
# spread v4 (block passes, ES rows zero off support) + FFT taper-group experiment
mkdir -p gpurun_out /tmp/ncu
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2n_c2.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2n_c5.log 2>&1
for g in 1 2 3; do NUS_FFT_GROUP=$g timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2n_c2_g$g.log 2>&1; done
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2n_c2f32.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py -q -x > gpurun_out/r2n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.log
NCU="ncu --set full --import-source on --clock-control none -c 1"
for kv in "stream_c5:spread_stream:--workload c5"; do
  name=${kv%%:*}; rest=${kv#*:}; re=${rest%%:*}; bargs=${rest#*:}
  timeout 600 $NCU -k regex:$re -s 2 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $bargs > gpurun_out/r2n_ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2n_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2n_${name}_src.csv.gz
done
