mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not 1d and not c2 and not c3_full" > gpurun_out/pytest_gen.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gen.log | grep -v Warn
timeout 900 python tools/gpu_general_stats.py c1 c4 c5 > gpurun_out/gen_stats.log 2>&1; echo stats=$?
cut -c1-900 gpurun_out/gen_stats.log
CR_DEBUG_STATS=1 timeout 900 python tools/gpu_general_stats.py c4 > gpurun_out/gen_stats_dbg.log 2>&1; echo dbg=$?
grep "\[cr\] dim" gpurun_out/gen_stats_dbg.log | cut -c1-400
