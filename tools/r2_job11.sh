# full GPU suite, smoke, default bench, reference arm, multi-rank functional check (gloo, 1 GPU)
mkdir -p gpurun_out
export LC_PARITY_LOG=gpurun_out/parity11.jsonl
rm -f $LC_PARITY_LOG
timeout -k 10 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest11.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/pytest11.log
timeout -k 10 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke11.log 2>&1; echo "smoke rc=$?"
timeout -k 10 900 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo "bench rc=$?"; tail -3 gpurun_out/bench11.err
LC_DIST_BACKEND=gloo timeout -k 10 600 python bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 --batched cfg3 > gpurun_out/bench11_g2.json 2> gpurun_out/bench11_g2.err; echo "g2 rc=$?"; tail -3 gpurun_out/bench11_g2.err
LC_DIST_BACKEND=gloo timeout -k 10 600 python bench.py --gpus 2 --config cfg5 --batched none --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench11_g2c5.json 2> gpurun_out/bench11_g2c5.err; echo "g2 cfg5 rc=$?"; tail -3 gpurun_out/bench11_g2c5.err
