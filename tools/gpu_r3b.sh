#!/bin/bash
# source-level ncu of the spreads: streaming (C2), two-group per-segment (C3 at 32 channels, C4 structure at 2^24)
mkdir -p gpurun_out /tmp/ncu
NCU="ncu --set full --import-source on --clock-control none -c 1"
cap() {  # name, kernel regex, env..., bench args in BARGS
  local name=$1 re=$2; shift 2
  timeout 900 env "$@" $NCU -k regex:$re -s 2 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $BARGS > gpurun_out/r3b_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r3b_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/${name}_sass.csv 2>&1
  gzip -c /tmp/ncu/${name}_sass.csv > gpurun_out/r3b_${name}_sass.csv.gz
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source cuda > /tmp/ncu/${name}_cuda.csv 2>&1
  gzip -c /tmp/ncu/${name}_cuda.csv > gpurun_out/r3b_${name}_cuda.csv.gz
}
BARGS="" cap stream_c2 spread_stream NUS_X=1
BARGS="--workload c3" cap c3 spread NUS_C3_CHANNELS=32
BARGS="--workload c4" cap c4 spread NUS_C4_LOG2N=24
ls -la gpurun_out/ | tail -20
