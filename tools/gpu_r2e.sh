#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2e_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_multi.log
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 5 > gpurun_out/r2e_bench.log 2>&1
timeout 900 python tools/diag/spline_c4.py 22 24 26 > gpurun_out/r2e_spline.log 2>&1
