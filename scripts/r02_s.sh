timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or small_class or k3" > gpurun_out/r02_s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_s_pytest.log
timeout 300 bash scripts/ab_ks.sh "5 15 31 33 45 53" twosucc > gpurun_out/r02_s_t.log 2>&1
CFG=c1 timeout 100 bash scripts/ab_ks.sh "31" twosucc >> gpurun_out/r02_s_t.log 2>&1
grep -E "passed|failed|rc=" gpurun_out/r02_s_pytest.log; cat gpurun_out/r02_s_t.log
