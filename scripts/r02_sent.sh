timeout 500 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity or forced or block_sort or spec_phase or golden" > gpurun_out/r02_sent_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_sent_pytest.log
timeout 300 bash scripts/ab_ks.sh "257 511" nosent > gpurun_out/r02_sent_ab.log 2>&1
CFG=c1 timeout 300 bash scripts/ab_ks.sh "101" nosent >> gpurun_out/r02_sent_ab.log 2>&1
CFG=c5 timeout 600 bash scripts/ab_ks.sh "100001" nosent >> gpurun_out/r02_sent_ab.log 2>&1
tail -2 gpurun_out/r02_sent_pytest.log; cat gpurun_out/r02_sent_ab.log
