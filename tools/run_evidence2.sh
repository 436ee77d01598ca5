# Evidence refresh: default bench line (cfg2 + cpu_baseline), reference arm, batched configs with the
# automatic engine and the level-pipelined engine for comparison.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/e_cfg2.json 2> gpurun_out/e_cfg2.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo ref rc=$?
for c in cfg3 cfg5; do
  for e in 0 1; do
    timeout 900 python bench.py --config $c --engine $e --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/e_${c}_e$e.json 2> gpurun_out/e_${c}_e$e.err; echo $c e$e rc=$?
  done
done
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/e_cfg4.json 2> gpurun_out/e_cfg4.err; echo cfg4 rc=$?
for f in gpurun_out/e_*.json; do python -c "
import json,sys; d=json.load(open('$f'))
rt=d.get('roofline_transform',{}); print('$f', d.get('impl','ours'), round(d['value']/1e9,2), 'Gcoef/s', round(d['ms_per_step'],4), 'ms/step frac', round(rt.get('frac',0),3), 'roof', d.get('roofline',{}).get('bound'), round(d.get('roofline',{}).get('frac',0) or 0,3), d['config'].get('kernel_cfg'))" 2>/dev/null || echo "$f unreadable"; done
