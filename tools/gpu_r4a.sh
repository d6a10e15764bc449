#!/bin/bash
# balanced pass B (fft_rows_crop_bal_kernel) against one row per CTA: C2 / C5 benches, parity tests with it forced on
mkdir -p gpurun_out
T=${TAG:-r4a}
for m in 0 1; do
  NUS_FFT_ROWS_BAL=$m timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/${T}_bal${m}_c2.log 2>&1
  NUS_FFT_ROWS_BAL=$m timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/${T}_bal${m}_c5.log 2>&1
done
timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 5 > gpurun_out/${T}_def_c2.log 2>&1
NUS_FFT_ROWS_BAL=1 timeout 1500 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py -m gpu -q -x > gpurun_out/${T}_tests_bal1.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_bal1.log
tail -3 gpurun_out/${T}_tests_bal1.log
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/${T}_*_c*.log')):
    try:
        d=json.loads(open(f).read().strip().split('\n')[-1])
        print(f.split('/')[-1], round(d['ms_per_step'],4), {k.replace('_kernel',''):round(v*1e3,1) for k,v in d['stages_ms'].items()})
    except Exception as e:
        print(f, 'ERR', e)
PY
