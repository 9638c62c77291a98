mkdir -p gpurun_out
python -c "import paper_2005_12692_b200" >/dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_level1 -s 3 -c 1 -o gpurun_out/l1 -f python tools/c2_time.py > gpurun_out/ncu_l1.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_l1.log
