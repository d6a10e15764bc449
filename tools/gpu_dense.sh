timeout 900 python -m pytest tests -m gpu -q -x -k "c3 or c4 or sweep" > gpurun_out/pytest_dense.log 2>&1; echo rc=$? >> gpurun_out/pytest_dense.log
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c4.log 2>&1
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep.json > gpurun_out/c5_sweep.log 2>&1
