# A/B of library variants on cfg4 (engine 3) with the range parity tests
cp paper_2411_00033_b200/liblegcheb.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  timeout 300 python -m pytest tests/test_gpu_tile.py tests/test_gpu_engines_sweep.py -q -x 2>&1 | tail -1
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$v cfg4', round(d['ms_per_step'],3), 'ms/step', [round(x,3) for x in d['kernel_ms']['leg2cheb']], round(d['roofline_transform']['frac'],3))" || tail -2 gpurun_out/ab.err
done
cp /tmp/lib_keep.so paper_2411_00033_b200/liblegcheb.so
