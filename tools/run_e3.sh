for c in cfg4 cfg3; do
for e in 3; do
timeout 900 python bench.py --config $c --engine $e --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b4.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json'))
print('$c e=$e', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['kernel_ms']['names'], round(d['roofline']['frac'],3))" || tail -3 gpurun_out/b.err
done
done
python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2411_00033_b200 import Plan
p=Plan(10**7,'leg2cheb',batch=64,device=torch.device('cuda',0),engine=3); print(p.kernel_info)"
