MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced" > gpurun_out/r02_msoa_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_msoa_chk.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or baseline_config_checksums and c1" > gpurun_out/r02_msoa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_msoa_pytest.log
CFG=c1 timeout 300 bash scripts/ab_ks.sh "101" nomsoa > gpurun_out/r02_msoa_t.log 2>&1
tail -2 gpurun_out/r02_msoa_chk.log; tail -2 gpurun_out/r02_msoa_pytest.log; cat gpurun_out/r02_msoa_t.log
