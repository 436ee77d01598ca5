timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "batched or batch_contiguous" 2>&1 | tail -3
for c in cfg3 cfg5; do for vt in 2 8; do
  timeout 600 python bench.py --config $c --vt $vt --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('$c vt=$vt', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'], 'rt', d['round_trip_einf'])" || tail -3 gpurun_out/b.err
done; done
