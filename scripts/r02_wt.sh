MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows" > gpurun_out/r02_wt_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_wt_chk.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows or baseline_config_checksums and (c1 or c2 or c3)" > gpurun_out/r02_wt_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_wt_pytest.log
timeout 300 bash scripts/ab_ks.sh "63 127 255 511 1023" wt > gpurun_out/r02_wt_t.log 2>&1
CFG=c1 timeout 100 bash scripts/ab_ks.sh "101" wt >> gpurun_out/r02_wt_t.log 2>&1
tail -2 gpurun_out/r02_wt_chk.log; tail -2 gpurun_out/r02_wt_pytest.log; cat gpurun_out/r02_wt_t.log
