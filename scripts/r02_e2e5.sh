timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "host or pipeline" > gpurun_out/r02_e2e5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_e2e5_pytest.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-check > gpurun_out/r02_e2e5_c5.log 2>&1
tail -2 gpurun_out/r02_e2e5_pytest.log; tail -1 gpurun_out/r02_e2e5_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])"
