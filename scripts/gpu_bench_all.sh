for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['config']['per_k_ms'])"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
