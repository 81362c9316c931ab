# Round evidence: GPU tests, bench (default + every config), launch list of the bench
# command, and one ncu --set full capture of each config-2 kernel.
set -x
timeout 1000 python -m pytest tests -q -m gpu -x > gpurun_out/ev_tests.log 2>&1; tail -1 gpurun_out/ev_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/ev_bench.log 2>&1; tail -1 gpurun_out/ev_bench.log
bash scripts/gpu_bench_all.sh > gpurun_out/ev_ball.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev_ncu1.log 2>&1
python scripts/profile_c2.py > gpurun_out/ev_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mf_ -s 0 -c 8 -o gpurun_out/ev_full -f \
    python scripts/profile_c2.py 3 31 255 1023 > gpurun_out/ev_ncu2.log 2>&1
tail -2 gpurun_out/ev_ncu2.log
