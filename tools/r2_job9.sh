mkdir -p gpurun_out
for g in 64 128; do
LC_UP_SPLIT=1 LC_UPB_GRID=$g timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl9_$g.txt 2>&1; sed -n 1,30p gpurun_out/tl9_$g.txt
done
