timeout 600 bash scripts/ab_ks.sh "255 1023" w1 w1b w8r8_2 > gpurun_out/r02_mexp.log 2>&1
cat gpurun_out/r02_mexp.log
