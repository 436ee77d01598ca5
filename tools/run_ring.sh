# cfg2: streaming-kernel ring geometry sweep (smaller rings let streaming CTAs co-reside with up CTAs)
timeout 600 python -m pytest tests/test_gpu_tile.py -q -x -k "staging" 2>&1 | tail -1
for sb in "3 3" "2 2" "1 3" "2 3" "1 2" "1 4"; do
  set -- $sb
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 3 --stage-blocks $1 --stages $2 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('cb=$1 nst=$2 cfg2', round(d['ms_per_step']*1e3/2,2), 'us/tr', [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -2 gpurun_out/ab.err
done
python -c "
import torch
from paper_2411_00033_b200 import Plan
for cb,nst in ((3,3),(2,2),(1,3),(2,3),(1,2),(1,4)):
    p=Plan(1000000,'leg2cheb',device=torch.device('cuda',0),stage_blocks=cb,stages=nst); ki=p.kernel_info
    print(cb,nst,ki['smem_stream'],ki['smem_up'],ki['stream_occ'],ki['kb'])
"
