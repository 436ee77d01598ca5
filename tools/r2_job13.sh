mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_partition.py -q -rf > gpurun_out/pytest13.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest13.log
timeout -k 10 300 python tools/part_times.py 1000000 1 2 4 8 > gpurun_out/part_times_1e6.txt 2>&1; cat gpurun_out/part_times_1e6.txt
timeout -k 10 300 python tools/part_times.py 10000000 1 2 4 8 > gpurun_out/part_times_1e7.txt 2>&1; cat gpurun_out/part_times_1e7.txt
