# A/B of library builds on engine-1 round trips (graph-replayed, tools/rt_time.py), alternating runs,
# then the engine-1 parity tests on the default build.  usage: bash tools/ab_down.sh liblegcheb_b.so [more .so]
LIBS="liblegcheb.so ${@:-liblegcheb_b.so}"
NS=${AB_NS:-"1000000 1048576 100000 10000000"}
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
  for lib in $LIBS; do
    for n in $NS; do
      echo "$rep $lib $n $(LC_LIB=$lib timeout 120 python tools/rt_time.py $n 1 400 2>&1 | tail -1)"
    done
  done
done | tee gpurun_out/ab/ab.txt
[ -n "$AB_NOTEST" ] || timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fig3.py -q -x 2>&1 | tail -3
