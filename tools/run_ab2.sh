cp paper_2411_00033_b200/liblegcheb.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$v cfg2', round(d['ms_per_step']*1e3/2,2), 'us/tr', [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])" || tail -2 gpurun_out/ab.err
done
cp /tmp/lib_keep.so paper_2411_00033_b200/liblegcheb.so
