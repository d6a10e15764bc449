#!/bin/bash
# round 2: rest of the GPU suite (after the C4 DPSS shape failure) + the 2^25/2^26 DPSS and spline diagnostics
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=15 --deselect "tests/test_gpu_fullsize.py::test_c4_full_2e26_vs_reference[es]" --deselect "tests/test_gpu_fullsize.py::test_c3_256x2e18_channels_fp32_vs_reference[es]" > gpurun_out/r2g_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_gpu.log
timeout 900 python tools/diag/spline_c4.py 22 24 26 > gpurun_out/r2g_spline.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_spline.log
timeout 1500 python tools/diag/dpss_2e26.py 24 25 26 > gpurun_out/r2g_dpss.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_dpss.log
