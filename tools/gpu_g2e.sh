timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_g2e.log 2>&1; echo rc=$? >> gpurun_out/pytest_g2e.log
NUS_C3_CHANNELS=32 timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c3_final.log 2>&1
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep.json > gpurun_out/c5_sweep.log 2>&1
