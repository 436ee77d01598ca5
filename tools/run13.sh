timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('cfg2', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step']*1e3/2,2), 'us/tr frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,4) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('cfg3', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 2>&1 | tail -2
