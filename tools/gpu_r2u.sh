#!/bin/bash
# validation after the reference-RNG inputs and the recurrence DPSS: smoke, bench (C2, C3 at 256 channels
# with its CPU baseline, C5), reference arm on C3, full GPU suite
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_smoke.log
timeout 400 python bench.py > gpurun_out/r2u_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench.log
timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/r2u_c3.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_c3.log
timeout 900 python bench.py --impl reference --workload c3 --steps 2 --warmup 3 > gpurun_out/r2u_c3ref.log 2>&1
timeout 400 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 > gpurun_out/r2u_c5.log 2>&1
timeout 3600 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r2u_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_gpu.log
