python tools/h0_var.py c4 2 3 2>&1 | tail -1 | cut -c60-140
python tools/h0_var.py c5 2 2 2>&1 | tail -1 | cut -c60-140
python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5b', d['stages_ms']['reduce_d1'])"
