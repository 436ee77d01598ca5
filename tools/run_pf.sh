for mb in 0 20 40 60 80; do
  LC_L2_PREFETCH_MB=$mb timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/pf.json 2>gpurun_out/pf.err
  python -c "
import json; d=json.load(open('gpurun_out/pf.json'))
print('pf $mb MB: cfg2', round(d['ms_per_step']*1e3/2,2), 'us/tr frac', round(d['roofline_transform']['frac'],3), [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])" || tail -2 gpurun_out/pf.err
done
