# full GPU check: tests, bench lines, ncu launch list + full captures (C2 top kernels, C5 k_filtration)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_all.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
tail -c 2500 gpurun_out/bench_c2.json
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; echo c4=$?
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1; echo c1=$?
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; echo c3=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reference_c2.json 2>&1; echo ref=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"k1_level1|k1_levels_coop" -s 4 -c 2 -o gpurun_out/prof_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1; echo c5=$?
python bench.py --config c5b --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5b.json 2>&1; echo c5b=$?
ncu --set full --clock-control none --import-source on -k regex:"k_filtration" -c 1 -o gpurun_out/prof_kf_c5 -f python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_kf.log 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:"k_filtration" -c 1 -o gpurun_out/prof_kf_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_kf4.log 2>&1; echo ncu4=$?
