for cfg in "2 6 3" "2 8 2" "8 4 2" "4 6 2"; do
set -- $cfg
timeout 900 python bench.py --config cfg4 --vt $1 --stage-blocks $2 --stages $3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b4.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b4.json'))
print('cfg4 vt=$1 cb=$2 nst=$3', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
