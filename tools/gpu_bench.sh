timeout 300 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/bench_c2f32.log 2>&1
NUS_KERNEL=gaussian timeout 300 python bench.py --no-cpu --steps 100 > gpurun_out/bench_c2_gauss.log 2>&1
