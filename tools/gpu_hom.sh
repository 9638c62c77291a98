mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "homology or topdim or fuzz or exhaustive_2x2 or cropped or k2_var or batched" > gpurun_out/pytest_hom.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_hom.log
python tools/h0_var.py c4 2 3 > gpurun_out/hom_c4.log 2>&1; echo c4=$?; cat gpurun_out/hom_c4.log | cut -c1-220
CR_K5_COHOM=1 python tools/h0_var.py c4 2 2 > gpurun_out/coh_c4.log 2>&1; echo c4c=$?; cat gpurun_out/coh_c4.log | cut -c1-220
python tools/h0_var.py c5 2 2 > gpurun_out/hom_c5.log 2>&1; echo c5=$?; cat gpurun_out/hom_c5.log | cut -c1-220
