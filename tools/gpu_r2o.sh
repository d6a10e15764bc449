#!/bin/bash
# streaming spread: interleaved work units (NUS_SPREAD_ILV) on C5 and C2; segment kernel reference
mkdir -p gpurun_out
for L in 1 2 4 8; do NUS_SPREAD_ILV=$L timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2o_c5_L$L.log 2>&1; done
for L in 1 2 4; do NUS_SPREAD_ILV=$L timeout 600 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 3 > gpurun_out/r2o_c2_L$L.log 2>&1; done
NUS_SPREAD=segment timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2o_c5_seg.log 2>&1
