CFG=c5 python scripts/profile_c2.py 100001 > gpurun_out/pl_plain.log 2>&1 && \
CFG=c5 ncu --set full --clock-control none --import-source on -k regex:"ml_unit|ml_walk|ml_tile|ml_merge" -s 0 -c 4 -o gpurun_out/prof_l5 -f \
    python scripts/profile_c2.py 100001 > gpurun_out/ncu_l5.log 2>&1
tail -1 gpurun_out/ncu_l5.log
