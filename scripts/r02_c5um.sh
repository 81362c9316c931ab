# ncu --set full of the large pipeline's pair merge and walk on config 5
CFG=c5 python scripts/profile_c2.py 100001 > gpurun_out/c5_plain.log 2>&1 && \
CFG=c5 ncu --set full --clock-control none --import-source on -k regex:"ml_unit_merge|ml_walk|ml_tile_sort" -c 3 -o gpurun_out/s4_c5um -f \
    python scripts/profile_c2.py 100001 > gpurun_out/c5_um.log 2>&1
tail -2 gpurun_out/c5_um.log
