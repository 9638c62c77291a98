# C4 stage diagnosis: launch list (per-kernel device time) + stage times under knobs
mkdir -p gpurun_out
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_plain.json 2>&1; echo plain=$?
CR_SMEM_BASINS=100000 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_smem.json 2>&1; echo smem=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo ncu=$?
