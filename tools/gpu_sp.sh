timeout 900 python -m pytest tests -m gpu -q -x -k "es or c2 or sweep or dense" > gpurun_out/pytest_sp.log 2>&1; echo rc=$? >> gpurun_out/pytest_sp.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_sp$i.log 2>&1; done
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 --workload c2f32 > gpurun_out/bench_sp32.log 2>&1
