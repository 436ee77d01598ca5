mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tile.py -x -q --timeout 300 > gpurun_out/pytest_tile.txt 2>&1; echo tile rc=$?
tail -3 gpurun_out/pytest_tile.txt
for c in cfg3 cfg5; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bt.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/bt.json'))
print('$c', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], round(d['roofline']['frac'],3), d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
