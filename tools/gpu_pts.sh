timeout 900 python -m pytest tests -m gpu -q -x -k "es or c2 or c3 or c4 or sweep" > gpurun_out/pytest_pts.log 2>&1; echo rc=$? >> gpurun_out/pytest_pts.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_pts$i.log 2>&1;
tail -1 gpurun_out/bench_pts$i.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['ms_per_step']*1e3,1), round(d['pipeline_roofline']['frac'],4), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})" >> gpurun_out/pts_summary.log; done
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 5 --no-cpu > gpurun_out/bench_c4_pts.log 2>&1
