#!/bin/bash
# streaming spread: parity tests + C2/C2f32/C5 bench against the per-segment kernel; C4 taper diag
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py tests/test_gpu_multi.py tests/test_gpu_tapers.py -q -x > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2i_c2.log 2>&1
NUS_SPREAD=segment timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2i_c2_seg.log 2>&1
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2i_c2f32.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2i_c5.log 2>&1
NUS_SPREAD_GROUPS=1 timeout 600 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2i_c3_g1.log 2>&1
timeout 900 python tools/diag/c4_tapers.py 22 24 26 > gpurun_out/r2i_c4tap.log 2>&1
