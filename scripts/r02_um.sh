timeout 500 python -m pytest tests/test_gpu_parity.py -q -x -k "large or block_sort or forced or golden" > gpurun_out/r02_um_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_um_pytest.log
CFG=c4 timeout 300 python scripts/time_ks.py 10001 > gpurun_out/r02_um_t.log 2>&1
CFG=c5 timeout 300 python scripts/time_ks.py 100001 >> gpurun_out/r02_um_t.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_checksums and (c4 or c5)" >> gpurun_out/r02_um_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_um_pytest.log
cat gpurun_out/r02_um_pytest.log | grep -E "passed|failed|rc="; cat gpurun_out/r02_um_t.log
