#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fft.py tests/test_gpu_tapers.py -q > gpurun_out/r2c_fft.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_fft.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/r2c_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_full.log
