timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "large or block_sort or spec_phase or forced" > gpurun_out/r02_soa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_soa_pytest.log
CFG=c4 timeout 300 bash scripts/ab_ks.sh "10001" nosoa > gpurun_out/r02_soa_ab.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_checksums and c4" >> gpurun_out/r02_soa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_soa_pytest.log
tail -4 gpurun_out/r02_soa_pytest.log; cat gpurun_out/r02_soa_ab.log
