#!/bin/bash
# fused pass A+B FFT: tests + C2/C2f32/C5/C3 benches (fused vs two-kernel); ncu of the stream v2 spread + fused FFT
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_fft.py -q -x -k "fused or c1_uses" > gpurun_out/r2l_fft.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_fft.log
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2l_c2.log 2>&1
NUS_FFT_FUSED=0 timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2l_c2_nofuse.log 2>&1
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2l_c2f32.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2l_c5.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2l_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_distributed.py tests/test_gpu_multi.py -q -x > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
NCU="ncu --set full --import-source on --clock-control none -c 1"
for kv in "stream_c2:spread_stream:" "fused_c2:fft_fused:" "stream_c5:spread_stream:--workload c5"; do
  name=${kv%%:*}; rest=${kv#*:}; re=${rest%%:*}; bargs=${rest#*:}
  timeout 600 $NCU -k regex:$re -s 2 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $bargs > gpurun_out/r2l_ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2l_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2l_${name}_src.csv.gz
done
