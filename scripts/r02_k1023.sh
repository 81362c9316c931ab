timeout 600 ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/r02_k1023 -f \
    python scripts/profile_c2.py 1023 > gpurun_out/k1023.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/r02_k255 -f \
    python scripts/profile_c2.py 255 > gpurun_out/k255.log 2>&1
tail -1 gpurun_out/k1023.log
