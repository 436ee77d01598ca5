timeout 300 python tools/timeline.py 1000000 leg2cheb 2>&1 | sed -n 1,22p
