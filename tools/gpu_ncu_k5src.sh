mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -c 1 -o gpurun_out/prof_k5_c4 -f python tools/h0_var.py c4 2 1 > gpurun_out/ncu_k5.log 2>&1; echo ncu=$?
