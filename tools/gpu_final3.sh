timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench_c2.log 2>&1
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/final_bench_c2f32.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/final_ncu_launch.log 2>&1
for k in spread_tc_kernel fft_rows_crop_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/final_$k -f python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/final_ncu_$k.log 2>&1
done
