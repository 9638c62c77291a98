mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apparent" -s 1 -c 1 -o gpurun_out/app -f python tools/k12_once.py c5 > gpurun_out/ncu_app.log 2>&1; echo ncu=$?
