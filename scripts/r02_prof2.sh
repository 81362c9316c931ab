CFG=c5 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ml_(tile|merge_pass)" -c 2 -o gpurun_out/r02_c5s -f \
    python scripts/profile_c2.py 100001 > gpurun_out/p2_c5s.log 2>&1
CFG=c5 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ml_(unit|walk)" -c 2 -o gpurun_out/r02_c5u -f \
    python scripts/profile_c2.py 100001 > gpurun_out/p2_c5u.log 2>&1
tail -1 gpurun_out/p2_c5s.log; tail -1 gpurun_out/p2_c5u.log; ls -la gpurun_out/
