# Evidence refresh: default bench line (cfg2 with both CPU baselines), reference arm, every config with
# the automatic engine, engine-1 comparisons, ncu launch lists and --set full summaries.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/e_cfg2.json 2> gpurun_out/e_cfg2.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo ref rc=$?
for c in cfg2b cfg3 cfg5 cfg4; do
  st=5; [ $c = cfg4 ] && st=3; [ $c = cfg2b ] && st=300
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/e_${c}.json 2> gpurun_out/e_${c}.err; echo $c rc=$?
done
for c in cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --config $c --engine 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/e_${c}_e1.json 2> gpurun_out/e_${c}_e1.err; echo $c e1 rc=$?
done
for f in gpurun_out/e_*.json; do python -c "
import json,sys; d=json.load(open('$f'))
rt=d.get('roofline_transform',{}); print('$f', d.get('impl','ours'), round(d['value']/1e9,3), 'Gcoef/s', round(d['ms_per_step'],4), 'ms/step frac', round(rt.get('frac',0),3), 'roof', d.get('roofline',{}).get('bound'), round(d.get('roofline',{}).get('frac',0) or 0,3), (d.get('config') or {}).get('kernel_cfg'))" 2>/dev/null || echo "$f unreadable"; done
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py $ARGS > gpurun_out/ncu_l2.log 2>&1; echo l2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_(up|stream|down)_kernel" -s 6 -c 3 -o gpurun_out/prof_cfg2 -f python bench.py $ARGS > gpurun_out/ncu_f2.log 2>&1; echo f2 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 $ARGS > gpurun_out/ncu_l3.log 2>&1; echo l3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_tile_kernel" -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 $ARGS > gpurun_out/ncu_f3.log 2>&1; echo f3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"lc_(up3|range)_kernel" -s 2 -c 2 -o gpurun_out/prof_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3 > gpurun_out/ncu_f4.log 2>&1; echo f4 rc=$?
