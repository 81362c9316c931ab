# usage: bash scripts/gpu_check.sh [pytest -m expr]
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/ -q -m "${1:-gpu}" > gpurun_out/t1.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED|^E  " gpurun_out/t1.log | head -60
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b1.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/b1.log
