timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in cfg2 cfg3 cfg4 cfg5; do
  st=300; [ $c != cfg2 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_$c.json 2>gpurun_out/f_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/f_$c.json'))
print('$c', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],4), 'ms/step frac', round(d['roofline_transform']['frac'],3), [round(x,4) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/f_$c.err
done
