# Evidence refresh after a tile/range-kernel change: cfg3, cfg5, cfg4 bench lines (+ engine-1 comparisons
# unchanged), cfg3 launch list and ncu of the tile kernel, ncu of the cfg4 up pass + range kernel
mkdir -p gpurun_out
for c in cfg3 cfg5 cfg4; do
  st=5; [ $c = cfg4 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/e_${c}.json 2> gpurun_out/e_${c}.err; echo $c rc=$?
done
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 $ARGS > gpurun_out/ncu_l3.log 2>&1; echo l3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 $ARGS > gpurun_out/ncu_f3.log 2>&1; echo f3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_(up3|range)_kernel" -s 2 -c 2 -o gpurun_out/prof_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3 > gpurun_out/ncu_f4.log 2>&1; echo f4 rc=$?
for c in cfg3 cfg5 cfg4; do python -c "
import json; d=json.load(open('gpurun_out/e_$c.json')); print('$c', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['roofline_transform']['frac'],3), round(d['roofline']['frac'],3), d['kernel_ms']['leg2cheb'], d['clocks'])"; done
