set -x
timeout 600 python bench.py > gpurun_out/final_bench_c2.log 2>&1
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/final_bench_c2f32.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/final_ncu_launch.log 2>&1
for k in spread_tc_kernel fft_cols_blk_kernel fft_rows_crop_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/final_$k -f python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/final_ncu_$k.log 2>&1
done
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep.json > gpurun_out/c5_sweep.log 2>&1
NUS_C4_LOG2N=26 timeout 1500 python bench.py --workload c4 --steps 5 --warmup 3 --e2e-steps 3 --no-cpu > gpurun_out/final_bench_c4_full.log 2>&1
