mkdir -p gpurun_out
CR_DEBUG_STATS=1 timeout 900 python tools/gpu_general_stats.py c4 c5 > gpurun_out/k5dbg.log 2>&1; echo a=$?
python bench.py --config c5b --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5b.json 2>&1; echo c5b=$?
