timeout 900 python -m pytest tests -m gpu -q -x -k "c3 or c4 or sweep" > gpurun_out/pytest_g2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g2.log
for w in c4 c3; do
timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_${w}_g2.log 2>&1
NUS_SPREAD_GROUPS=1 timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_${w}_g1.log 2>&1
done
