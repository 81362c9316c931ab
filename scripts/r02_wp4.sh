MF_B200_LIB=$PWD/_variants/wp4chk/libmedfilt_b200.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "random_parity and not large or golden or forced or rows" > gpurun_out/r02_wp4_chk.log 2>&1; echo "rc=$?" >> gpurun_out/r02_wp4_chk.log
MF_B200_LIB=$PWD/_variants/wp4w1m5/libmedfilt_b200.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "baseline_config_checksums and c2_k1023" > gpurun_out/r02_wp4_g.log 2>&1; echo "rc=$?" >> gpurun_out/r02_wp4_g.log
timeout 400 bash scripts/ab_ks.sh "513 767 1023" wp4w1m5 wp4w1m4 wp4w2m3 > gpurun_out/r02_wp4_t.log 2>&1
tail -2 gpurun_out/r02_wp4_chk.log; tail -2 gpurun_out/r02_wp4_g.log; cat gpurun_out/r02_wp4_t.log
