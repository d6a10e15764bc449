# launch list + one full capture per stage kernel (C2 fp64, default ES window)
set -x
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ncu_pre.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ncu_launch.log 2>&1
for k in spread_tc_kernel fft_cols_blk_kernel fft_rows_crop_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/full_$k -f python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
