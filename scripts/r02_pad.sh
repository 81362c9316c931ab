timeout 500 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows or small_class" > gpurun_out/r02_pad_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pad_pytest.log
timeout 300 bash scripts/ab_ks.sh "33 63 101 127 255 1023" nopad > gpurun_out/r02_pad_ab.log 2>&1
tail -2 gpurun_out/r02_pad_pytest.log; cat gpurun_out/r02_pad_ab.log
