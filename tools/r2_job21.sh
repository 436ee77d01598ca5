mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py -q -x -rf > gpurun_out/pytest21.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest21.log
for n in 1000000 10000000; do timeout -k 10 300 python tools/part_times.py $n 1 2 4 8 --up > gpurun_out/part_up_$n.txt 2>&1; tail -1 gpurun_out/part_up_$n.txt; done
timeout -k 10 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/split_check.py 1000000 up 2>&1 | grep rank | tail -4
