for cfg in "3 3" "3 2" "4 2" "5 2" "4 3"; do
  set -- $cfg
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --stage-blocks $1 --stages $2 --e2e-steps 3 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('cb=$1 nst=$2', round(d['ms_per_step']*1e3/2,2), 'us/transform; kernels', [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || echo fail $cfg
done
