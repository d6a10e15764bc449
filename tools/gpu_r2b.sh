#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fft.py tests/test_gpu_tapers.py -q > gpurun_out/r2b_fft.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_fft.log
