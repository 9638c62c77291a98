#!/bin/bash
# One GPU session: bench (default C5b) -> ncu launch list -> ncu --set full of k_filtration and
# k_reduce -> GPU tests.  Usage (on the box, via gpurun): bash tools/gpu_session.sh OUTDIR [tests]
set -u
O=${1:-gpurun_out/sess}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches_c5b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5 \
  > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_filtration -c 1 -f \
  -o $O/kf_c5b python tools/run_once.py c5b > $O/ncu_kf.log 2>&1; echo "ncu kf rc=$?"
if [ "${2:-}" = "tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 $O/pytest_gpu.log
fi
