CFG=c1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/r02_c1b -f \
    python scripts/profile_c2.py 101 > gpurun_out/c1p.log 2>&1
tail -1 gpurun_out/c1p.log
