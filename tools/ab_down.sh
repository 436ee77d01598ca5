# A/B of two library builds on engine-1 round trips (graph-replayed, tools/rt_time.py), alternating runs,
# then the engine-1 parity tests on the default build.  usage: bash tools/ab_down.sh liblegcheb_b.so
B=${1:-liblegcheb_b.so}
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
  for lib in liblegcheb.so $B; do
    for n in 1000000 1048576 100000 10000000; do
      echo "$rep $lib $n $(LC_LIB=$lib timeout 120 python tools/rt_time.py $n 1 400 2>&1 | tail -1)"
    done
  done
done | tee gpurun_out/ab/ab.txt
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fig3.py -q -x 2>&1 | tail -3
