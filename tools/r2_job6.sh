# split up pass: parity (engine 1), A/B bench, upb grid sweep, timeline
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_memsafety.py tests/test_gpu_engines_sweep.py tests/test_gpu_boundary.py -q -rf -x > gpurun_out/pytest6.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest6.log
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
for sp in 0 1; do
  LC_UP_SPLIT=$sp timeout 300 $B > gpurun_out/b6_split$sp.json 2>gpurun_out/b6_split$sp.err; echo "split=$sp rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/b6_split$sp.json'));print('split $sp', d['ms_per_step'], d['step_ms'], d['roofline_transform']['frac'], d['kernel_ms']['names'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']])"
done
for g in 16 64 128; do
  LC_UP_SPLIT=1 LC_UPB_GRID=$g timeout 300 $B > gpurun_out/b6_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b6_g$g.json'));print('upb grid $g', d['ms_per_step'], d['roofline_transform']['frac'])"
done
LC_UP_SPLIT=1 timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl6.txt 2>&1; echo "tl rc=$?"; head -30 gpurun_out/tl6.txt
