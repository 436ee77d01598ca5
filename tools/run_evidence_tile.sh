# Evidence refresh for the per-tile kernel (engine 2): cfg3 and cfg5 bench lines, cfg3 launch list and ncu --set full
mkdir -p gpurun_out
for c in cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/e_${c}.json 2> gpurun_out/e_${c}.err; echo $c rc=$?
done
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 $ARGS > gpurun_out/ncu_l3.log 2>&1; echo l3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 $ARGS > gpurun_out/ncu_f3.log 2>&1; echo f3 rc=$?
for f in gpurun_out/e_cfg3.json gpurun_out/e_cfg5.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['roofline_transform']['frac'],3), round(d['roofline']['frac'],3), d['clocks'])"; done
