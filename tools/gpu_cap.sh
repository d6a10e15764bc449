#!/bin/bash
# source-level ncu capture of kernels of one bench command.
# usage: TAG=r3g KERNELS="fft_cols_blk fft_rows_crop" BARGS="--workload c2" bash tools/gpu_cap.sh
mkdir -p gpurun_out /tmp/ncu
T=${TAG:-cap}
NCU="ncu -f --set full --import-source on --clock-control none -c 1"
for re in $KERNELS; do
  name=${re}${SUFFIX}
  timeout 900 $NCU -k regex:$re -s ${SKIP:-3} -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $BARGS > gpurun_out/${T}_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/${T}_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass | gzip -c > gpurun_out/${T}_${name}_sass.csv.gz
done
ls -la gpurun_out | grep ${T}_
