#!/bin/bash
# A/B: streaming spread at 4 CTAs/SM (168 registers) vs 5 CTAs/SM (128 registers, spills); larger
# normalisation chunks at full C4 (setup)
mkdir -p gpurun_out
for w in c2 c5; do timeout 400 python bench.py --workload $w --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2v_${w}_4cta.log 2>&1; done
cp paper_2407_01943_b200/lib/libnus_b200.so /tmp/lib_main.so; cp build_alt/libnus_b200.so paper_2407_01943_b200/lib/libnus_b200.so
for w in c2 c5; do timeout 400 python bench.py --workload $w --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2v_${w}_5cta.log 2>&1; done
cp /tmp/lib_main.so paper_2407_01943_b200/lib/libnus_b200.so
NUS_C4_LOG2N=26 timeout 1200 python bench.py --workload c4 --no-cpu --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/r2v_c4full.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_c4full.log
timeout 900 python -m pytest tests/test_gpu_tapers.py tests/test_gpu_distributed.py -q -x > gpurun_out/r2v_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests.log
