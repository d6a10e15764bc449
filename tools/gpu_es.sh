timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "es or c1 or c2 or sweep or c5 or c3" > gpurun_out/pytest_es.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_es.log
timeout 300 python bench.py --no-cpu --steps 100 > gpurun_out/bench_es.log 2>&1
timeout 300 python bench.py --no-cpu --steps 100 --workload c2f32 > gpurun_out/bench_es_f32.log 2>&1
