timeout 600 python -m pytest tests/test_gpu_tile.py -q -x 2>&1 | tail -2
python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2411_00033_b200 import Plan
p=Plan(4096,'leg2cheb',batch=4096,device=torch.device('cuda',0)); print(p.kernel_info)"
cp paper_2411_00033_b200/liblegcheb.so /tmp/keep.so
for v in MINB3 MINB2; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  for c in cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$v $c', round(d['ms_per_step'],3), 'ms/step', [round(x,3) for x in d['kernel_ms']['leg2cheb']], round(d['roofline_transform']['frac'],3))" || tail -2 gpurun_out/ab.err
  done
done
cp /tmp/keep.so paper_2411_00033_b200/liblegcheb.so
