mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_mm.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_mm.log
python tools/h0_var.py c1 1 6 > gpurun_out/mm_c1.log 2>&1; tail -2 gpurun_out/mm_c1.log | cut -c1-200
python tools/h0_var.py c4 2 3 > gpurun_out/mm_c4.log 2>&1; tail -1 gpurun_out/mm_c4.log | cut -c1-200
python tools/h0_var.py c5 2 2 > gpurun_out/mm_c5.log 2>&1; tail -1 gpurun_out/mm_c5.log | cut -c1-200
