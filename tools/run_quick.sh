# quick GPU check: parity suite + cfg2/cfg3 bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.txt
for i in 1 2; do
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('cfg2', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step']*1e3/2,2), 'us/tr frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,4) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b3.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b3.json'))
print('cfg3', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
