timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/h0_var.py c4 2 3 2>&1 | tail -1 | cut -c1-180
python tools/h0_var.py c5 2 2 2>&1 | tail -1 | cut -c1-180
