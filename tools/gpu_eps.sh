for e in 1e-3 1e-4 1e-6; do
timeout 300 python bench.py --no-cpu --steps 50 --eps $e > gpurun_out/bench_eps_$e.log 2>&1
done
