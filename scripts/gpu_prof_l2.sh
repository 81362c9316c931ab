CFG=c5 python scripts/profile_c2.py 100001 > gpurun_out/pl_plain.log 2>&1 && \
CFG=c5 ncu --set full --clock-control none --import-source on -k regex:"ml_unit|ml_walk" -s 0 -c 2 -o gpurun_out/prof_l5b -f \
    python scripts/profile_c2.py 100001 > gpurun_out/ncu_l5b.log 2>&1
tail -1 gpurun_out/ncu_l5b.log
