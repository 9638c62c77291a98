mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "1d or c2 or host or edge or golden or sin or batched_1d" > gpurun_out/pytest_1d.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_1d.log
timeout 300 python tools/c2_time.py > gpurun_out/c2_time.log 2>&1; echo time=$?
cat gpurun_out/c2_time.log
