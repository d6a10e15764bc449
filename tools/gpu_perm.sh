timeout 900 python -m pytest tests -m gpu -q -x -k "es or c2 or c1 or dense or sweep" > gpurun_out/pytest_perm.log 2>&1; echo rc=$? >> gpurun_out/pytest_perm.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_perm$i.log 2>&1;
tail -1 gpurun_out/bench_perm$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['ms_per_step']*1e3,1), round(d['pipeline_roofline']['frac'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})" >> gpurun_out/perm_summary.log; done
