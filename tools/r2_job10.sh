mkdir -p gpurun_out
export LC_UP_SPLIT=0
for ks in 3 2; do
LC_UP_KSUB=$ks timeout -k 10 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "single_vector or cfg or back_to_back or batched" > gpurun_out/pytest10_$ks.log 2>&1; echo "ksub=$ks pytest rc=$?"; tail -2 gpurun_out/pytest10_$ks.log
done
B="python bench.py --config cfg2 --batched none --no-cpu-baseline --steps 3000 --warmup 50 --e2e-steps 3"
for ks in 6 5 4 3 2; do
  LC_UP_KSUB=$ks timeout 300 $B > gpurun_out/b10_k$ks.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b10_k$ks.json'));print('ksub $ks', d['ms_per_step'], d['roofline_transform']['frac'], [round(x*1e3,1) for x in d['kernel_ms']['leg2cheb']], d['round_trip_einf']['device'])"
done
LC_UP_KSUB=3 timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl10.txt 2>&1; sed -n 1,22p gpurun_out/tl10.txt
