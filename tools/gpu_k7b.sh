timeout 900 python -m pytest tests -m gpu -x -q -k "batched or c3 or lifetime or edge" 2>&1 | tail -2
python tools/k7_time.py 2>&1 | tail -2
CR_TOP_REDUCE=1 python tools/k7_time.py 2>&1 | tail -1
