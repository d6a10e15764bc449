#!/bin/bash
# round 2 (re-entry): verify the last commit on the B200 — smoke, full GPU suite, C2 bench, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r2f_gpu.txt 2>&1
nproc >> gpurun_out/r2f_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_smoke.log
timeout 300 python bench.py --steps 200 --warmup 20 > gpurun_out/r2f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_bench.log
timeout 300 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 > gpurun_out/r2f_bench_f32.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --no-cpu --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/r2f_ncu.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/r2f_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_gpu.log
