timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
NUS_DPSS_PROF=1 timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
