mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k7_image" -c 1 -o gpurun_out/prof_k7 -f python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_k7.log 2>&1; echo ncu=$?
