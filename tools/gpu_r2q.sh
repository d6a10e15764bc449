#!/bin/bash
# packed point records + auto interleave: tests + C2/C2f32/C5 benches
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2q_c2.log 2>&1
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2q_c2f32.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2q_c5.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py tests/test_gpu_multi.py tests/test_gpu_fft.py tests/test_gpu_dropin.py -q -x > gpurun_out/r2q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_tests.log
