for k in 2 3 4 6 8; do
  timeout 300 python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 200 --warmup 10 --e2e-steps 200 --e2e-streams $k > gpurun_out/e2e_$k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e_$k.json'));print('streams $k', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
timeout 300 python tools/pcie_bw.py 2>&1 | tail -5
