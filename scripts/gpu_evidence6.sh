# Round evidence at the end of the third session: GPU tests, bench, launch list of the bench command,
# ncu --set full of the k = 3 kernel, smoke().
set -x
timeout 1000 python -m pytest tests -q -m gpu -x > gpurun_out/ev6_tests.log 2>&1; tail -1 gpurun_out/ev6_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev6_smoke.log 2>&1; tail -1 gpurun_out/ev6_smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/ev6_bench.log 2>&1; tail -1 gpurun_out/ev6_bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev6_ref.log 2>&1; tail -1 gpurun_out/ev6_ref.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/ev6_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ev6_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mf_med3 -s 0 -c 1 -o gpurun_out/ev6_med3 -f \
    python scripts/profile_c2.py 3 > gpurun_out/ev6_ncu2.log 2>&1
tail -1 gpurun_out/ev6_ncu2.log
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/ev6_bench_$c.log 2>&1; tail -1 gpurun_out/ev6_bench_$c.log | cut -c1-200; done
bash scripts/gpu_launches.sh c5 100001 ev6_launches_c5
bash scripts/gpu_launches.sh c4 10001 ev6_launches_c4
