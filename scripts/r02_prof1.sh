# ncu --set full with source: S at k=31 (c2), M f64 k=101 (c1), the large pipeline on c4
set -x
python scripts/profile_c2.py 31 > gpurun_out/p1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_small -s 1 -c 1 -o gpurun_out/r02_s31 -f \
    python scripts/profile_c2.py 31 > gpurun_out/p1_s31.log 2>&1
CFG=c1 ncu --set full --clock-control none --import-source on -k regex:mf_medium -s 1 -c 1 -o gpurun_out/r02_c1 -f \
    python scripts/profile_c2.py 101 > gpurun_out/p1_c1.log 2>&1
CFG=c4 python scripts/profile_c2.py 10001 > gpurun_out/p1_c4plain.log 2>&1 && \
CFG=c4 ncu --set full --clock-control none --import-source on -k regex:ml_ -c 8 -o gpurun_out/r02_c4 -f \
    python scripts/profile_c2.py 10001 > gpurun_out/p1_c4.log 2>&1
CFG=c4 python scripts/time_ks.py 10001 > gpurun_out/p1_c4time.log 2>&1
CFG=c1 python scripts/time_ks.py 101 > gpurun_out/p1_c1time.log 2>&1
tail -2 gpurun_out/p1_c4.log
