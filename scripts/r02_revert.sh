timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02_revert_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_revert_pytest.log
CFG=c5 timeout 300 python scripts/time_ks.py 100001 > gpurun_out/r02_revert_t.log 2>&1
timeout 300 python scripts/time_ks.py 255 1023 >> gpurun_out/r02_revert_t.log 2>&1
tail -2 gpurun_out/r02_revert_pytest.log; cat gpurun_out/r02_revert_t.log
