mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_reduce" -s 0 -c 1 -o gpurun_out/k5 -f python tools/k12_once.py c4 > gpurun_out/ncu_k5.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_k5.log
