#!/bin/bash
# streaming spread: interleave on C5 (K 7 and 15), C3 (K 9) single-group streaming vs two-group segment kernel
mkdir -p gpurun_out
for L in 16 32; do NUS_SPREAD_ILV=$L timeout 600 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r2p_c5_L$L.log 2>&1; done
NUS_C5_K=15 timeout 600 python bench.py --workload c5 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2p_c5k15_g2.log 2>&1
for L in 1 8; do NUS_C5_K=15 NUS_SPREAD_GROUPS=1 NUS_SPREAD_ILV=$L timeout 600 python bench.py --workload c5 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2p_c5k15_L$L.log 2>&1; done
for L in 1 4 8; do NUS_SPREAD_GROUPS=1 NUS_SPREAD_ILV=$L timeout 600 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/r2p_c3_L$L.log 2>&1; done
NUS_C4_LOG2N=24 timeout 900 python bench.py --workload c4 --no-cpu --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r2p_c4_g2.log 2>&1
NUS_C4_LOG2N=24 NUS_SPREAD_GROUPS=1 NUS_SPREAD_ILV=8 timeout 900 python bench.py --workload c4 --no-cpu --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r2p_c4_L8.log 2>&1
