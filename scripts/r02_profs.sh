# ncu --set full with source of the small kernel at k = 31 and the k = 3 kernel (config 2)
python scripts/profile_c2.py 31 3 > gpurun_out/ps_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_small -s 1 -c 1 -o gpurun_out/s4_s31 -f \
    python scripts/profile_c2.py 31 > gpurun_out/ps_31.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mf_med3 -s 1 -c 1 -o gpurun_out/s4_t3 -f \
    python scripts/profile_c2.py 3 > gpurun_out/ps_3.log 2>&1
tail -2 gpurun_out/ps_3.log
