mkdir -p gpurun_out
cp paper_2411_00033_b200/liblegcheb.so /tmp/keep.so
for v in VOL NV; do
  cp exp/lib_$v.so paper_2411_00033_b200/liblegcheb.so
  for c in "129 8" "200 13" "1000 9" "4096 8"; do
    timeout 60 python tools/tile_one.py $c; echo "$v $c rc=$?"
  done
done
cp exp/lib_NV.so paper_2411_00033_b200/liblegcheb.so
timeout 240 compute-sanitizer --tool synccheck python tools/tile_one.py 1000 9 2>&1 | tail -15; echo sync rc=$?
cp /tmp/keep.so paper_2411_00033_b200/liblegcheb.so
