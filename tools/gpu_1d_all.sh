bash tools/gpu_1d.sh
bash tools/gpu_ncu_l1.sh
