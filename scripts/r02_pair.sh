MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "large or golden or forced" > gpurun_out/r02_pair_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pair_chk.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "large or golden or forced or phase" > gpurun_out/r02_pair_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pair_pytest.log
CFG=c4 timeout 300 bash scripts/ab_ks.sh "10001" nopair > gpurun_out/r02_pair_t.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_checksums and c4" >> gpurun_out/r02_pair_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pair_pytest.log
grep -E "passed|failed|rc=|Error" gpurun_out/r02_pair_chk.log | tail -3; grep -E "passed|failed|rc=" gpurun_out/r02_pair_pytest.log; cat gpurun_out/r02_pair_t.log
