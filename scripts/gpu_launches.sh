# launch list (per-kernel device times) for one config: bash scripts/gpu_launches.sh CFG "ks" name
CFG=$1 python scripts/profile_c2.py $2 > gpurun_out/lp_plain.log 2>&1 && \
CFG=$1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/$3.csv python scripts/profile_c2.py $2 > gpurun_out/$3.log 2>&1
tail -1 gpurun_out/$3.log
