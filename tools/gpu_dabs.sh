timeout 900 python -m pytest tests -m gpu -x -q -k "topdim or fuzz or cropped or batched or homology or edge or c5 or lifetime" 2>&1 | tail -2
python tools/h0_var.py c5 2 2 2>&1 | tail -1 | cut -c60-160
python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
