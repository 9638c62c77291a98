python tools/k7_time.py 2>&1 | tail -3
CR_TOP_REDUCE=1 python tools/k7_time.py 2>&1 | tail -1
