cp paper_2411_00033_b200/liblegcheb.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  echo "== $v"; timeout 600 python tools/range_batches.py 2000000
done
cp /tmp/lib_keep.so paper_2411_00033_b200/liblegcheb.so
timeout 600 python -m pytest tests/test_gpu_tile.py tests/test_gpu_engines_sweep.py -q -x 2>&1 | tail -1
