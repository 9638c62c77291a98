mkdir -p gpurun_out
python tools/h0_var.py c5 2 6 > gpurun_out/h0var_c5_2.log 2>&1; echo b=$?
python tools/h0_var.py c4 2 8 > gpurun_out/h0var_c4_2.log 2>&1; echo c=$?
python tools/h0_var.py c1 1 8 > gpurun_out/h0var_c1_1.log 2>&1; echo d=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_all.log
