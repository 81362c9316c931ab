# quick GPU loop: non-slow parity tests, then the config-2 per-k timings
timeout 1500 python -m pytest tests/ -q -m "gpu and not slow" -x > gpurun_out/tq.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED|^E  " gpurun_out/tq.log | head -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], d['value'], d['config']['per_k_ms'])"
if [ -n "$E2E" ]; then
  python scripts/pcie_probe.py
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', d['e2e'])"
fi
