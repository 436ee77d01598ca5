for vt in 2 4 8; do
timeout 900 python bench.py --config cfg4 --vt $vt --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b4.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json'))
print('cfg4 vt=$vt', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
