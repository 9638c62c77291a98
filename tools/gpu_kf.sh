# fused K1+K2 (k_filtration): parity + C4/C5 stage times + ncu on the kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "k2_variants or fuzz or exhaustive_2x2 or topdim or cropped or golden or edge" > gpurun_out/kf_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/kf_pytest.log
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/kf_c5.json 2>&1; echo c5=$?
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/kf_c4.json 2>&1; echo c4=$?
CR_K12_OLD=1 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/kf_c4_old.json 2>&1; echo c4old=$?
ncu --set full --clock-control none --import-source on -k regex:"k_filtration" -c 1 -o gpurun_out/prof_kf_c5 -f python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_kf.log 2>&1; echo ncu=$?
