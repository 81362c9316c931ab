CFG=c5 python scripts/time_ks.py 100001 > gpurun_out/c5p_time.log 2>&1
CFG=c5 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ml_ -c 12 -o gpurun_out/r02_c5 -f \
    python scripts/profile_c2.py 100001 > gpurun_out/c5p_ncu.log 2>&1
tail -2 gpurun_out/c5p_ncu.log; cat gpurun_out/c5p_time.log
