for cfg in "" "NUS_PDL=1" "NUS_PDL=1 NUS_PDL_TAIL=1" "NUS_PDL=1 NUS_PDL_TAIL=1 NUS_PDL_SPREAD_NOWAIT=1"; do
  env $cfg timeout 300 python bench.py --no-cpu --steps 200 --e2e-steps 20 > gpurun_out/pdl.log 2>&1
  echo "$cfg :: $(python -c "
import json
d=json.loads(open('gpurun_out/pdl.log').read().strip().splitlines()[-1])
print(round(d['ms_per_step']*1e3,1), 'frac', round(d['pipeline_roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,2))
")" >> gpurun_out/pdl_summary.log
done
