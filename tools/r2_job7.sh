mkdir -p gpurun_out
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
for db in 0 1; do
  LC_UP_SPLIT=0 LC_DOWN_BULK=$db timeout 300 $B > gpurun_out/b7_db$db.json 2>gpurun_out/b7_db$db.err; echo "db=$db rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/b7_db$db.json'));print('down_bulk $db', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf'])"
done
for k in 5 7; do
  LC_UP_SPLIT=0 timeout 300 $B --up-subtree $k > gpurun_out/b7_k$k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b7_k$k.json'));print('kup $k', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])"
done
LC_UP_SPLIT=0 timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl7.txt 2>&1; sed -n 1,20p gpurun_out/tl7.txt
