MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so timeout 500 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity or golden or forced or block_sort or spec_phase or rows" > gpurun_out/r02_clamp_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_clamp_chk.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity or golden or forced or block_sort or spec_phase or rows or baseline_config_checksums" > gpurun_out/r02_clamp_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_clamp_pytest.log
CFG=c5 timeout 300 bash scripts/ab_ks.sh "100001" clamp > gpurun_out/r02_clamp_t.log 2>&1
CFG=c4 timeout 300 bash scripts/ab_ks.sh "10001" clamp >> gpurun_out/r02_clamp_t.log 2>&1
CFG=c1 timeout 100 bash scripts/ab_ks.sh "101" clamp >> gpurun_out/r02_clamp_t.log 2>&1
timeout 100 bash scripts/ab_ks.sh "257 511" clamp >> gpurun_out/r02_clamp_t.log 2>&1
tail -2 gpurun_out/r02_clamp_chk.log; tail -2 gpurun_out/r02_clamp_pytest.log; cat gpurun_out/r02_clamp_t.log
