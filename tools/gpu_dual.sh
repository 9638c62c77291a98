mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_all.log | grep -v Warn
timeout 900 python tools/gpu_general_stats.py c1 c4 c5 > gpurun_out/gen_stats.log 2>&1; echo stats=$?
grep -o '^c[0-9]\|"reduce_d[12]": [0-9.]*\|"h0": [0-9.]*\|"columns": \[[0-9, ]*\]\|"rounds": \[[0-9, ]*\]\|"wall_s": [0-9.]*' gpurun_out/gen_stats.log | tr '\n' ' '; echo
CR_TOP_REDUCE=1 timeout 900 python tools/gpu_general_stats.py c1 > gpurun_out/gen_stats_red.log 2>&1
grep -o '^c[0-9]\|"reduce_d[12]": [0-9.]*\|"wall_s": [0-9.]*' gpurun_out/gen_stats_red.log | tr '\n' ' '; echo
