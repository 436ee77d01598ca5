mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest26.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest26.log
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
timeout 300 $B > gpurun_out/b26.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b26.json'));print('cfg2', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf']['device'])"
