# hash rank recovery: parity under the checked build first (bounded by timeout), then A/B timings
export MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows" > gpurun_out/r02_hash_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_hash_chk.log
unset MF_B200_LIB
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows" > gpurun_out/r02_hash_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_hash_pytest.log
timeout 300 bash scripts/ab_ks.sh "33 63 101 127 255 511 1023" nohash > gpurun_out/r02_hash_ab.log 2>&1
tail -2 gpurun_out/r02_hash_chk.log; tail -2 gpurun_out/r02_hash_pytest.log; cat gpurun_out/r02_hash_ab.log
