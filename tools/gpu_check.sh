set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/time_1d_phases.py > gpurun_out/phases.log 2>&1; echo phases=$?
cat gpurun_out/phases.log
