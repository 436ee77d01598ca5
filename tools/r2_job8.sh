mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_memsafety.py tests/test_gpu_engines_sweep.py -q -rf -x > gpurun_out/pytest8.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest8.log
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
for sp in 0 1; do
  LC_UP_SPLIT=$sp timeout 300 $B > gpurun_out/b8_split$sp.json 2>gpurun_out/b8_split$sp.err; echo "split=$sp rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/b8_split$sp.json'));print('split $sp', d['ms_per_step'], d['roofline_transform']['frac'], d['kernel_ms']['names'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf'])"
done
for g in 32 128; do
  LC_UP_SPLIT=1 LC_UPB_GRID=$g timeout 300 $B > gpurun_out/b8_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b8_g$g.json'));print('upb grid $g', d['ms_per_step'], d['roofline_transform']['frac'])"
done
LC_UP_SPLIT=1 timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl8.txt 2>&1; sed -n 1,20p gpurun_out/tl8.txt
