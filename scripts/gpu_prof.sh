# ncu evidence: launch list of the bench command, then a full capture of each c2 kernel.
set -x
python scripts/profile_c2.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_c2.py > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_ -s 1 -c 8 -o gpurun_out/prof_c2 -f \
    python scripts/profile_c2.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
