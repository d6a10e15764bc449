#!/bin/bash
# round 2: own FFT at every grid size + full GPU suite + smoke + C2 bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/r2a_gpu.txt 2>&1
free -g >> gpurun_out/r2a_gpu.txt; nproc >> gpurun_out/r2a_gpu.txt
timeout 1500 python -m pytest tests/test_gpu_fft.py -q -x > gpurun_out/r2a_fft.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_fft.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fft.py > gpurun_out/r2a_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_gpu.log
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/r2a_bench.log 2>&1
