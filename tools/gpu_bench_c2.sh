set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?
tail -c 3000 gpurun_out/bench_c2.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k1_deaths -s 2 -c 1 -o gpurun_out/prof_c2_deaths python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out
