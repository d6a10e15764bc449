timeout 900 python -m pytest tests -m gpu -q -x -k "sweep or c4 or c3" > gpurun_out/pytest_k31.log 2>&1; echo rc=$? >> gpurun_out/pytest_k31.log
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep.json > gpurun_out/c5_sweep.log 2>&1
