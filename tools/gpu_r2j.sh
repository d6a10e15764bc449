#!/bin/bash
# ncu --set full of the spread kernels (streaming vs per-segment) on C2 and C5, source-level;
# only the text exports come back (the reports exceed gpurun's 64 MiB)
mkdir -p gpurun_out /tmp/ncu
NCU="ncu --set full --import-source on --clock-control none -c 1"
cap() {  # name, kernel regex, env..., bench args
  local name=$1 re=$2; shift 2
  timeout 600 env "$@" $NCU -k regex:$re -s 2 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $BARGS > gpurun_out/r2j_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2j_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/${name}_src.csv 2>&1
  gzip -c /tmp/ncu/${name}_src.csv > gpurun_out/r2j_${name}_src.csv.gz
}
BARGS="" cap stream_c2 spread_stream NUS_X=1
BARGS="--workload c5" cap stream_c5 spread_stream NUS_X=1
BARGS="--workload c5" cap seg_c5 spread_tc NUS_SPREAD=segment
BARGS="--workload c3" cap c3 spread NUS_X=1
ls -la gpurun_out/ | tail -20
