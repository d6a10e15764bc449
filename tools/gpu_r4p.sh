#!/bin/bash
# end-of-round-2 evidence after the two-tile-wide layout blocks: smoke, default bench, reference arm, fp32 / C5 / C3 / full C4, launch list, ncu of the C2 kernels (GPU suite: r4o)
mkdir -p gpurun_out /tmp/ncu
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r4p_smoke.log
timeout 400 python bench.py > gpurun_out/r4p_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4p_bench.log
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r4p_ref.log 2>&1
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/r4p_c2f32.log 2>&1
timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 > gpurun_out/r4p_c5.log 2>&1
timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 > gpurun_out/r4p_c3.log 2>&1
NUS_C4_LOG2N=26 timeout 1200 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/r4p_c4full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r4p_launches.csv python bench.py --no-cpu --steps 3 --warmup 3 --e2e-steps 3 > gpurun_out/r4p_ncu_launch.log 2>&1
NCU="ncu -f --set full --import-source on --clock-control none -c 1"
for kv in "spread_stream_kernel:spread_stream" "fft_cols_blk_kernel:fft_cols_blk" "fft_rows_crop_kernel:fft_rows_crop"; do
  name=${kv%%:*}; re=${kv#*:}
  timeout 600 $NCU -k regex:$re -s 3 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r4p_ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r4p_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/r4p_${name}_raw.csv 2>&1
done
