mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile.py -x -q --timeout 300 > gpurun_out/pytest_tile.txt 2>&1; echo tile rc=$?
tail -15 gpurun_out/pytest_tile.txt
for e in 2 1; do
timeout 600 python bench.py --config cfg3 --engine $e --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b3e.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b3e.json'))
print('cfg3 engine=$e', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['roofline']['frac'], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
