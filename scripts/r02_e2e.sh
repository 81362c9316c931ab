set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "host or rows or pipeline" > gpurun_out/r02_e2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_e2e_pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02_e2e_bench.log 2>&1
tail -3 gpurun_out/r02_e2e_pytest.log
