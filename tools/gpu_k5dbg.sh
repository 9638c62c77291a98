mkdir -p gpurun_out
CR_DEBUG_STATS=1 timeout 900 python tools/gpu_general_stats.py c5 > gpurun_out/k5dbg5.log 2>&1; echo a=$?
