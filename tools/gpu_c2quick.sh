mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "1d or c2 or host or edge or golden or sin or batched_1d" > gpurun_out/pytest_1d.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_1d.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c2q.json 2>&1; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_c2q.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['stages_ms'],d['e2e']['ms_per_step'])"
