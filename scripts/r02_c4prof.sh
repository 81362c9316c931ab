CFG=c4 python scripts/profile_c2.py 10001 > gpurun_out/c4p_plain.log 2>&1 && \
CFG=c4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ml_ -c 8 -o gpurun_out/r02_c4b -f \
    python scripts/profile_c2.py 10001 > gpurun_out/c4p_ncu.log 2>&1
tail -2 gpurun_out/c4p_ncu.log
