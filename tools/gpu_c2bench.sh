bash tools/gpu_1d.sh
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'],d['e2e']['ms_per_step'])"
