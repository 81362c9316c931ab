# Evidence for the bench line: plain run, launch list of the same command, and one
# --set full capture of each config-2 kernel (the dominant one feeds roofline.traffic).
set -x
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev_ncu1.log 2>&1
python scripts/profile_c2.py > gpurun_out/ev_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_ -s 4 -c 4 -o gpurun_out/ev_full -f \
    python scripts/profile_c2.py > gpurun_out/ev_ncu2.log 2>&1
tail -2 gpurun_out/ev_ncu2.log
