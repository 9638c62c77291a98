CR_DEBUG_STATS=1 timeout 900 python tools/gpu_general_stats.py c4 c5 2>&1 | grep "\[cr\]" 
