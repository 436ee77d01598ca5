for v in NO_M2L NO_BAND NO_M2LDLC_EXP_NO_BAND; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('$v', round(d['ms_per_step']*1e3/2,2), 'us/tr', 'kernels', [round(x,4) for x in d['kernel_ms']['leg2cheb']])" || tail -2 gpurun_out/b.err
done
