timeout 900 python -m pytest tests -m gpu -q -x -k "es or c1 or c2 or sweep or c3 or c4" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_quick.log 2>&1
