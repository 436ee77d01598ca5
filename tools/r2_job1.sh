# round 2, job 1: full GPU test suite with the parity log, smoke, compute-sanitizer per engine
mkdir -p gpurun_out
export LC_PARITY_LOG=gpurun_out/parity.jsonl
rm -f $LC_PARITY_LOG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout -k 10 1500 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout -k 10 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for tool in memcheck racecheck synccheck; do
  for e in 1 2 3; do
    timeout -k 10 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $e > gpurun_out/san_${tool}_e$e.log 2>&1
    echo "$tool engine $e rc=$?"; tail -3 gpurun_out/san_${tool}_e$e.log
  done
done
