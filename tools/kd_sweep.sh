B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
for k in 3 4 5 6; do
  timeout 300 $B --subtree $k > gpurun_out/b27_k$k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b27_k$k.json'));print('kd $k', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf']['device'], d['config']['kernel_cfg'])"
done
