timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "k3 or golden or random_parity and (k0 or 3-)" > gpurun_out/r02_med3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_med3_pytest.log
timeout 300 bash scripts/ab_ks.sh "3" med3old > gpurun_out/r02_med3_t.log 2>&1
CFG=c1 timeout 100 bash scripts/ab_ks.sh "3" med3old >> gpurun_out/r02_med3_t.log 2>&1
tail -2 gpurun_out/r02_med3_pytest.log; cat gpurun_out/r02_med3_t.log
