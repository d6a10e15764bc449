#!/bin/bash
# layout blocks of 2^lw pass-A tiles (NUS_FFT_LW): C2 / C5 / C5 at K = 15 / C4's structure at 2^24, parity with it on
mkdir -p gpurun_out
for lw in 0 1 2 3; do
  NUS_FFT_LW=$lw timeout 300 python bench.py --no-cpu --steps 200 --warmup 20 --e2e-steps 3 > gpurun_out/r4m_lw${lw}_c2.log 2>&1
  NUS_FFT_LW=$lw timeout 300 python bench.py --workload c5 --no-cpu --steps 100 --warmup 10 --e2e-steps 3 > gpurun_out/r4m_lw${lw}_c5.log 2>&1
  NUS_FFT_LW=$lw NUS_C5_K=15 timeout 300 python bench.py --workload c5 --no-cpu --steps 50 --warmup 5 --e2e-steps 2 > gpurun_out/r4m_lw${lw}_c5k15.log 2>&1
  NUS_FFT_LW=$lw NUS_C4_LOG2N=24 timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/r4m_lw${lw}_c4s.log 2>&1
done
NUS_FFT_LW=3 timeout 1500 python -m pytest tests/test_gpu_mtnufft.py tests/test_gpu_nufft.py tests/test_gpu_fft.py -m gpu -q -x > gpurun_out/r4m_tests_lw3.log 2>&1; echo rc=$? >> gpurun_out/r4m_tests_lw3.log; tail -2 gpurun_out/r4m_tests_lw3.log
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/r4m_lw*.log')):
    try:
        d=json.loads([l for l in open(f).read().strip().split('\n') if l.startswith('{')][-1])
        print(f.split('/')[-1], round(d['ms_per_step'],4), {k.replace('_kernel',''):round(v*1e3,1) for k,v in d['stages_ms'].items()})
    except Exception as e:
        print(f, 'ERR', e)
PY
