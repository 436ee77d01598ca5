# A/B of library variants on cfg4 (engine 3) and cfg2 (engine 1), parity first
cp paper_2411_00033_b200/liblegcheb.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  timeout 300 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py tests/test_gpu_engines_sweep.py -q -x 2>&1 | tail -1
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$v cfg4', round(d['ms_per_step'],3), 'ms/step', [round(x,3) for x in d['kernel_ms']['leg2cheb']], round(d['roofline_transform']['frac'],3))" || tail -2 gpurun_out/ab.err
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$v cfg2', round(d['ms_per_step']*1e3/2,2), 'us/tr', [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])" || tail -2 gpurun_out/ab.err
done
cp /tmp/lib_keep.so paper_2411_00033_b200/liblegcheb.so
