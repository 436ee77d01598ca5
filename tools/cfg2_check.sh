# engine-1 parity subset, the cfg2 bench line and the phase timeline (debug build)
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_memsafety.py tests/test_gpu_partition.py tests/test_gpu_engines_sweep.py tests/test_gpu_boundary.py -q -x -rf > gpurun_out/pytest_c2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c2.log
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
timeout 300 $B > gpurun_out/b_c2.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_c2.json'));print('cfg2', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf']['device'])"
timeout 300 python tools/timeline.py 1000000 leg2cheb 2>&1 | sed -n 14,22p
