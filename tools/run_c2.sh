timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for c in cfg2 cfg2b; do
  timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c2.json 2>gpurun_out/c2.err
  python -c "
import json; d=json.load(open('gpurun_out/c2.json'))
print('$c', round(d['ms_per_step']*1e3/2,2), 'us/tr frac', round(d['roofline_transform']['frac'],3), [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])" || tail -2 gpurun_out/c2.err
done
