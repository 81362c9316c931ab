timeout 600 python -m pytest tests -m gpu -q > gpurun_out/r02_phase_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_phase_pytest.log
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_phase_c5.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_phase_c2.log 2>&1
tail -2 gpurun_out/r02_phase_pytest.log; tail -1 gpurun_out/r02_phase_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['phases'], d['ms_per_step'])"
