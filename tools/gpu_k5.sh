mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not 1d and not c2 and not c3_full" > gpurun_out/pytest_gen.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gen.log | grep -v Warn
for m in 4096 65536; do
  CR_K5_MCAP=$m timeout 900 python tools/gpu_general_stats.py c4 c5 > gpurun_out/gen_stats_$m.log 2>&1; echo stats=$?
  python - $m <<'PY'
import json,sys
for l in open(f"gpurun_out/gen_stats_{sys.argv[1]}.log"):
    if l[:2] in ("c4","c5"):
        n,j=l.split(" ",1); d=json.loads(j); print(sys.argv[1], n, {k:round(v,2) for k,v in d["stages"].items()}, d["rounds"])
PY
done
CR_DEBUG_STATS=1 timeout 900 python tools/gpu_general_stats.py c4 2>&1 | grep "attempt\|per add\|phase-A" | head -12
