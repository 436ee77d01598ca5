mkdir -p gpurun_out
timeout -k 10 900 python bench.py --config cfg4 --batched none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench14_cfg4.json 2> gpurun_out/bench14_cfg4.err; echo "cfg4 rc=$?"; tail -2 gpurun_out/bench14_cfg4.err
LC_DIST_BACKEND=gloo timeout -k 10 600 python bench.py --gpus 2 --split-vector --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 --batched none > gpurun_out/bench14_split.json 2> gpurun_out/bench14_split.err; echo "split rc=$?"; tail -3 gpurun_out/bench14_split.err
python -c "
import json
for f in ['bench14_cfg4.json','bench14_split.json']:
    d=json.loads(open('gpurun_out/'+f).read().strip().splitlines()[-1]); print(f, d['n_gpus'], d['value'], d['ms_per_step'], d['roofline_transform']['frac'], d['round_trip_einf'], d['e2e']['value'], d['config']['workload'])
"
