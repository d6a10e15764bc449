for m in 0 48; do
NUS_SPREAD_DENSE_MIN=$m timeout 900 python tools/c5_sweep.py --k 15 31 --out gpurun_out/c5_g2d_$m.json > gpurun_out/c5_g2d_$m.log 2>&1
NUS_SPREAD_DENSE_MIN=$m NUS_C3_CHANNELS=32 timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c3_$m.log 2>&1
done
