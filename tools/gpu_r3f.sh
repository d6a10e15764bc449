#!/bin/bash
# after the ring spread: parity subset, C4 structure (two-group per-segment vs two streaming launches), C5 at K=15,
# source-level captures of the streaming spread on C2 and C5
mkdir -p gpurun_out /tmp/ncu
T=r3f
timeout 1500 python -m pytest tests/test_gpu_nufft.py tests/test_gpu_mtnufft.py tests/test_gpu_es.py tests/test_gpu_multi.py tests/test_gpu_distributed.py -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
NUS_C4_LOG2N=24 timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/${T}_c4.log 2>&1
NUS_SPREAD_GROUPS=1 NUS_C4_LOG2N=24 timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/${T}_c4_stream2.log 2>&1
NUS_C5_K=15 timeout 300 python bench.py --workload c5 --no-cpu --steps 50 --warmup 5 --e2e-steps 2 > gpurun_out/${T}_c5k15.log 2>&1
NUS_SPREAD_GROUPS=1 NUS_C5_K=15 timeout 300 python bench.py --workload c5 --no-cpu --steps 50 --warmup 5 --e2e-steps 2 > gpurun_out/${T}_c5k15_stream2.log 2>&1
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/${T}_c*.log')):
    try:
        d=json.loads(open(f).read().strip().split('\n')[-1])
        print(f.split('/')[-1], round(d['ms_per_step'],4), {k.replace('_kernel',''):round(v*1e3,1) for k,v in d['stages_ms'].items()}, d.get('setup_ms',{}).get('total'))
    except Exception as e:
        print(f, 'ERR', e)
PY
NCU="ncu --set full --import-source on --clock-control none -c 1"
cap() {  # name, kernel regex, bench args in BARGS
  local name=$1 re=$2
  timeout 900 $NCU -k regex:$re -s 3 -o /tmp/ncu/$name python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 $BARGS > gpurun_out/${T}_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/${T}_${name}_details.csv 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass | gzip -c > gpurun_out/${T}_${name}_sass.csv.gz
}
BARGS="" cap stream_c2 spread_stream
BARGS="--workload c5" cap stream_c5 spread_stream
