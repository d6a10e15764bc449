NUS_SPREAD_XSORT=1 timeout 600 python -m pytest tests -m gpu -q -x -k "c2 or c1" > gpurun_out/pytest_xs.log 2>&1; echo rc=$? >> gpurun_out/pytest_xs.log
for v in 0 1 0 1; do NUS_SPREAD_XSORT=$v timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_xs$v.log 2>&1;
tail -1 gpurun_out/bench_xs$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('xsort $v', round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()}, d['gpu_launches'])" >> gpurun_out/xs_summary.log; done
