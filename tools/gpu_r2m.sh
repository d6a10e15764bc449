#!/bin/bash
# spread v3 (4-point steps): tests + benches + ncu source of the spread at C2 and C5; sharded bench modes at world 1
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py tests/test_gpu_multi.py tests/test_gpu_fft.py -q -x > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2m_c2.log 2>&1
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2m_c2f32.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2m_c5.log 2>&1
NUS_SPREAD_GROUPS=1 timeout 600 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2m_c3_g1.log 2>&1
NUS_KERNEL=gaussian timeout 600 python bench.py --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2m_c2_gauss.log 2>&1
NUS_C3_CHANNELS=16 timeout 600 python bench.py --shard channels --steps 10 --warmup 3 > gpurun_out/r2m_shard_ch.log 2>&1
timeout 600 python bench.py --shard tapers --steps 10 --warmup 3 > gpurun_out/r2m_shard_tp.log 2>&1
NUS_C4_LOG2N=22 timeout 600 python bench.py --shard samples --steps 10 --warmup 3 > gpurun_out/r2m_shard_sm.log 2>&1
NCU="ncu --set full --import-source on --clock-control none -c 1"
for kv in "stream_c2:spread_stream:" "stream_c5:spread_stream:--workload c5"; do
  name=${kv%%:*}; rest=${kv#*:}; re=${rest%%:*}; bargs=${rest#*:}
  timeout 600 $NCU -k regex:$re -s 2 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $bargs > gpurun_out/r2m_ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2m_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2m_${name}_src.csv.gz
done
