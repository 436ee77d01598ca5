timeout -k 10 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/split_check.py 1000000 2>&1 | grep -v OMP | tail -12
