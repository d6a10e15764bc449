#!/bin/bash
# ring-phase streaming spread: parity subset, stage times on C2 / C2 fp32 / C5 / C3 (two-group vs two streaming
# launches), instruction count of the C2 spread, source-level capture of the two-group per-segment spread on C3
mkdir -p gpurun_out /tmp/ncu
T=${TAG:-r3c}
timeout 1200 python -m pytest tests/test_gpu_nufft.py tests/test_gpu_mtnufft.py tests/test_gpu_es.py tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
timeout 300 python bench.py --no-cpu > gpurun_out/${T}_c2.log 2>&1
timeout 300 python bench.py --workload c2f32 --no-cpu > gpurun_out/${T}_c2f32.log 2>&1
timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 > gpurun_out/${T}_c5.log 2>&1
NUS_C3_CHANNELS=32 timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 > gpurun_out/${T}_c3.log 2>&1
NUS_SPREAD_GROUPS=1 NUS_C3_CHANNELS=32 timeout 300 python bench.py --workload c3 --no-cpu --steps 50 --warmup 5 > gpurun_out/${T}_c3_stream2.log 2>&1
NUS_C4_LOG2N=24 timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 > gpurun_out/${T}_c4.log 2>&1
NUS_SPREAD_GROUPS=1 NUS_C4_LOG2N=24 timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 > gpurun_out/${T}_c4_stream2.log 2>&1
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/${T}_c*.log')):
    try:
        d=json.loads(open(f).read().strip().split('\n')[-1])
        print(f, round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, 'pipe', round(d['pipeline_roofline']['frac'],3))
    except Exception as e:
        print(f, 'ERR', e)
PY
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:spread_stream -s 3 -c 1 --clock-control none python bench.py --no-cpu --steps 2 --warmup 3 --e2e-steps 1 2>&1 | grep -E "inst_executed|time_duration|dram__|issue_active" 
if [ -n "$CAP" ]; then
NCU="ncu --set full --import-source on --clock-control none -c 1"
NUS_C3_CHANNELS=32 timeout 900 $NCU -k regex:spread_tc -s 2 -o /tmp/ncu/c3tc python bench.py --workload c3 --no-cpu --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/${T}_cap_c3.log 2>&1
ncu -i /tmp/ncu/c3tc.ncu-rep --page details --csv > gpurun_out/${T}_c3tc_details.csv 2>&1
ncu -i /tmp/ncu/c3tc.ncu-rep --page source --csv --print-source sass | gzip -c > gpurun_out/${T}_c3tc_sass.csv.gz
fi
