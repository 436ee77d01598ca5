for cfg in "0 0" "5 0" "7 0" "0 5" "0 7" "5 5" "7 7"; do
  set -- $cfg
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 --up-subtree $1 --subtree $2 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('kup=$1 kd=$2', round(d['ms_per_step']*1e3/2,2), 'us/tr', [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -2 gpurun_out/sw.err
done
