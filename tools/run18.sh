cp exp/lib-DLC_EXP_NOCOARSEWAIT.so paper_2411_00033_b200/liblegcheb_dbg.so
timeout 300 python tools/timeline.py 1000000 leg2cheb > gpurun_out/tl_nc.txt 2>&1
