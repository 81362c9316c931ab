CFG=c5 timeout 900 bash scripts/ab_ks.sh "100001" bl0 bl1 bl3 > gpurun_out/r02_knobs.log 2>&1
CFG=c4 timeout 300 bash scripts/ab_ks.sh "10001" minb4 bl1 >> gpurun_out/r02_knobs.log 2>&1
cat gpurun_out/r02_knobs.log
