mkdir -p gpurun_out
for vt in 2 4 8; do
timeout 600 python bench.py --config cfg3 --vt $vt --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b3_$vt.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b3_$vt.json'))
print('cfg3 vt=$vt', round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],3), 'ms/step', 'frac', round(d['roofline_transform']['frac'],3), 'kernels', [round(x,3) for x in d['kernel_ms']['leg2cheb']], [round(x,3) for x in d['kernel_ms']['cheb2leg']], d['config']['kernel_cfg'])" || tail -3 gpurun_out/b.err
done
python tools/prof_cfg.py 4096 4096 2 leg2cheb 2 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 3 -c 3 -o gpurun_out/prof_b3_vt2 -f python tools/prof_cfg.py 4096 4096 2 leg2cheb 2 > gpurun_out/ncu_b3.log 2>&1
echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 3 -c 3 -o gpurun_out/prof_b3_vt8 -f python tools/prof_cfg.py 4096 4096 2 leg2cheb 8 > gpurun_out/ncu_b3_8.log 2>&1
echo ncu8 rc=$?
