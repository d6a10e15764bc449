#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py tests/test_gpu_fft.py -q -x > gpurun_out/r2d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_tests.log
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 5 > gpurun_out/r2d_bench.log 2>&1
bash tools/gpu_il.sh
timeout 1500 python tools/diag/dpss_2e26.py 25 26 > gpurun_out/r2d_dpss.log 2>&1
