# Evidence refresh after a range-kernel change: all GPU tests, cfg4 bench line, ncu of the cfg4 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/e_cfg4.json 2> gpurun_out/e_cfg4.err; echo cfg4 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_(up3|range)_kernel" -s 2 -c 2 -o gpurun_out/prof_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3 > gpurun_out/ncu_f4.log 2>&1; echo f4 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/e_cfg4.json')); print('cfg4', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['roofline_transform']['frac'],3), round(d['roofline']['frac'],3), d['kernel_ms']['leg2cheb'], d['kernel_ms']['cheb2leg'], d['clocks'])"
timeout 300 python tools/range_batches.py 2000000
