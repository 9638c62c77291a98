timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
CR_SMEM_BASINS=56000 timeout 900 python -m pytest tests -m gpu -x -q -k "topdim or fuzz or exhaustive or golden or c1 or c4_cropped" 2>&1 | tail -1
timeout 900 python tools/gpu_general_stats.py c1 c4 c5 2>&1 | grep -o '^c[0-9]\|"h0": [0-9.]*\|"reduce_d[12]": [0-9.]*\|"rounds": \[[0-9, ]*\]\|"wall_s": [0-9.]*' | tr '\n' ' '; echo
