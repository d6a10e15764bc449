#!/bin/bash
# DPSS recurrence tests + full C4 (2^26) setup and spectrum with the new DPSS path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tapers.py -q -x > gpurun_out/r2t_tapers.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_tapers.log
NUS_C4_LOG2N=26 timeout 1200 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/r2t_c4full.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_c4full.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4 or dpss" > gpurun_out/r2t_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_full.log
