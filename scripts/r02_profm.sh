# ncu --set full with source of the medium kernel at k = 255 and k = 1023 (config 2)
python scripts/profile_c2.py 255 1023 > gpurun_out/pm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/s4_m255 -f \
    python scripts/profile_c2.py 255 > gpurun_out/pm_255.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/s4_m1023 -f \
    python scripts/profile_c2.py 1023 > gpurun_out/pm_1023.log 2>&1
tail -2 gpurun_out/pm_1023.log
