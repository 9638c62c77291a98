mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batched or c3 or c4 or c5 or fuzz or topdim or k2_var or exhaustive" > gpurun_out/pytest_k5.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_k5.log
python bench.py --config c5b --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5b.json 2>&1; echo c5b=$?
python tools/h0_var.py c4 2 3 > gpurun_out/h0var_c4_2.log 2>&1; echo c4=$?
