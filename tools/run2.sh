mkdir -p gpurun_out
timeout 120 python -c "
import torch, numpy as np, sys
sys.path.insert(0,'.')
from paper_2411_00033_b200 import Plan
from lc_inputs import vector
import oracle
dev=torch.device('cuda',0)
for n in [5, 100, 1024, 4096, 65536, 1000000]:
    x=torch.from_numpy(vector('sign_over_j1', n, 0, 0)).to(dev)
    p=Plan(n,'leg2cheb',device=dev); q=Plan(n,'cheb2leg',device=dev)
    y=p.execute(x); z=q.execute(y); torch.cuda.synchronize()
    print(n, 'rt', float((z-x).abs().max()/x.abs().max()), p.desc['vt'], p.desc['subtree'], flush=True)
" > gpurun_out/quick.txt 2>&1; echo quick rc=$?; cat gpurun_out/quick.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench rc=$?
tail -3 gpurun_out/bench_cfg2.err
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_cfg2.txt 2>&1; echo tl rc=$?
