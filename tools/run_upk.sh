# cfg4: subtree depth of the persistent up pass (engine 3)
for k in 3 2 1; do
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 --up-subtree $k > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('kup=$k cfg4', round(d['ms_per_step'],3), 'ms/step', [round(x,3) for x in d['kernel_ms']['leg2cheb']], round(d['roofline_transform']['frac'],3))" || tail -2 gpurun_out/ab.err
done
