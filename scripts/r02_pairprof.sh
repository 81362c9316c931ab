CFG=c4 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:ml_pair" -c 1 -o gpurun_out/r02_pair -f \
    python scripts/profile_c2.py 10001 > gpurun_out/pp.log 2>&1
tail -1 gpurun_out/pp.log
