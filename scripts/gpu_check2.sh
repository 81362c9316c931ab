nvidia-smi --query-gpu=name --format=csv,noheader
timeout 2400 python -m pytest tests/ -q -m "${1:-gpu}" -x > gpurun_out/t1.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED|^E  " gpurun_out/t1.log | head -30
for c in c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'])"; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['value'], d['config']['per_k_ms'])"
