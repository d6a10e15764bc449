timeout 900 python -m pytest tests -m gpu -q -x -k "c4 or normalisation" > gpurun_out/pytest_c4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c4.log
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c5.log 2>&1
NUS_C3_CHANNELS=32 timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c3.log 2>&1
