#!/bin/bash
# A/B of alternate library builds (build_alt/<v>/libnus_b200.so against the in-tree one): stage times of
# C2 / C2 fp32 / C5 (+ C3 at 32 channels with EXTRA=1).  usage: VARIANTS="v1 v3" TAG=r3d bash tools/gpu_variants.sh
mkdir -p gpurun_out
T=${TAG:-var}
LIB=paper_2407_01943_b200/lib/libnus_b200.so
cp $LIB /tmp/libnus_b200_v0.so
for v in v0 $VARIANTS; do
  if [ $v = v0 ]; then cp /tmp/libnus_b200_v0.so $LIB; else cp build_alt/$v/libnus_b200.so $LIB; fi
  timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 3 > gpurun_out/${T}_${v}_c2.log 2>&1
  timeout 300 python bench.py --workload c2f32 --no-cpu --steps 200 --warmup 20 --e2e-steps 3 > gpurun_out/${T}_${v}_c2f32.log 2>&1
  timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/${T}_${v}_c5.log 2>&1
  if [ -n "$EXTRA" ]; then
    NUS_C3_CHANNELS=32 timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/${T}_${v}_c3.log 2>&1
    NUS_SPREAD_GROUPS=1 NUS_C3_CHANNELS=32 timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 --e2e-steps 3 > gpurun_out/${T}_${v}_c3s2.log 2>&1
  fi
done
cp /tmp/libnus_b200_v0.so $LIB
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/${T}_v*.log')):
    try:
        d=json.loads(open(f).read().strip().split('\n')[-1])
        print(f.split('/')[-1], round(d['ms_per_step'],4), {k.replace('_kernel',''):round(v*1e3,1) for k,v in d['stages_ms'].items()})
    except Exception as e:
        print(f, 'ERR', e)
PY
