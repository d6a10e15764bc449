python -c "
import torch
p=torch.cuda.get_device_properties(0)
print('l2', p.L2_cache_size)
" > gpurun_out/l2.log 2>&1
for mb in 0 32 56 80; do
if [ $mb = 0 ]; then unset NUS_L2_PERSIST_MB; else export NUS_L2_PERSIST_MB=$mb; fi
timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/bench_l2_$mb.log 2>&1
tail -1 gpurun_out/bench_l2_$mb.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('mb $mb', round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['stages_ms'].items()})" >> gpurun_out/l2.log
done
