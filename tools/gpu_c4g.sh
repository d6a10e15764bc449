for g in 2 1; do
NUS_SPREAD_GROUPS=$g timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c4_$g.log 2>&1
done
