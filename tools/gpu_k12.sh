mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not 1d and not c2 and not c3_full" > gpurun_out/pytest_gen.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gen.log | grep -v Warn
bash tools/gpu_ncu_k12.sh
