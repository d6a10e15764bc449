NUS_SPREAD_GROUPS=2 timeout 600 python -m pytest tests -m gpu -q -x -k "c4 or c3 or sweep" > gpurun_out/pytest_g2b.log 2>&1; echo rc=$? >> gpurun_out/pytest_g2b.log
for g in 2 1; do
NUS_SPREAD_GROUPS=$g timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c4_$g.log 2>&1
NUS_SPREAD_GROUPS=$g timeout 900 python tools/c5_sweep.py --k 15 --out gpurun_out/c5_k15_$g.json > gpurun_out/c5_k15_$g.log 2>&1
done
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_c2_g.log 2>&1
