#!/bin/bash
# streaming spread v2 (phase ring, zero-filled ES rows, pipelined steps): tests + benches; C4 shape diag
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_es.py tests/test_gpu_distributed.py tests/test_gpu_multi.py -q -x > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2k_c2.log 2>&1
timeout 600 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/r2k_c2f32.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2k_c5.log 2>&1
NUS_SPREAD_GROUPS=1 timeout 600 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2k_c3_g1.log 2>&1
NUS_KERNEL=gaussian timeout 600 python bench.py --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2k_c2_gauss.log 2>&1
timeout 1200 python tools/diag/c4_shape.py 26 15 > gpurun_out/r2k_c4shape.log 2>&1
