#!/bin/bash
# re-entry check: smoke, default bench, C2 fp32 / C5 / C3(32) stage times, GPU suite
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_smoke.log
timeout 400 python bench.py > gpurun_out/r3a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_bench.log
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/r3a_c2f32.log 2>&1
timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 > gpurun_out/r3a_c5.log 2>&1
NUS_C3_CHANNELS=32 timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 > gpurun_out/r3a_c3.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r3a_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_gpu.log
tail -3 gpurun_out/r3a_gpu.log
