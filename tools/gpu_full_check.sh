# the full GPU suite, smoke, one default bench line and the multi-rank paths run functionally on one GPU (gloo)
mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_full.log
timeout -k 10 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
LC_DIST_BACKEND=gloo timeout -k 10 600 python bench.py --gpus 2 --config cfg5 --batched none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/g2_cfg5.json 2> gpurun_out/g2_cfg5.err; echo "g2 cfg5 rc=$?"
LC_DIST_BACKEND=gloo timeout -k 10 600 python bench.py --gpus 2 --split-vector --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 --batched cfg3 > gpurun_out/g2_split.json 2> gpurun_out/g2_split.err; echo "g2 split rc=$?"
python -c "
import json
for f in ['g2_cfg5.json','g2_split.json']:
    d=json.loads(open('gpurun_out/'+f).read().strip().splitlines()[-1]); print(f, d['n_gpus'], d['value'], d['round_trip_einf'], d.get('passes_ms'), d.get('batched',{}).get('round_trip_einf'))
"
