mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "c4 or c5 or fuzz or exhaustive or golden or topdim or k2" > gpurun_out/pytest_k5.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_k5.log
timeout 900 python tools/gpu_general_stats.py c4 c5 > gpurun_out/gen_stats.log 2>&1; echo stats=$?
grep -o '^c[0-9]\|"reduce_d[12]": [0-9.]*\|"h0": [0-9.]*' gpurun_out/gen_stats.log | tr '\n' ' '; echo
CR_K5_NOCACHE=1 timeout 900 python tools/gpu_general_stats.py c4 > gpurun_out/gen_stats_np.log 2>&1; echo stats=$?
grep -o '^c[0-9]\|"reduce_d[12]": [0-9.]*' gpurun_out/gen_stats_np.log | tr '\n' ' '; echo
