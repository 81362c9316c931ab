timeout 500 python -m pytest tests/test_gpu_parity.py -q -x -k "large or block_sort or forced or golden" > gpurun_out/r02_soa32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_soa32_pytest.log
CFG=c5 timeout 600 bash scripts/ab_ks.sh "100001" nosoa32 > gpurun_out/r02_soa32_t.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_checksums and (c4 or c5)" >> gpurun_out/r02_soa32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_soa32_pytest.log
grep -E "passed|failed|rc=" gpurun_out/r02_soa32_pytest.log; cat gpurun_out/r02_soa32_t.log
