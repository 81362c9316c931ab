# Round evidence, third session: GPU tests, bench (default + every config), launch lists of
# the large-k configs, one ncu --set full capture of the large-k pipeline's kernels (c5).
set -x
timeout 1000 python -m pytest tests -q -m gpu -x > gpurun_out/ev3_tests.log 2>&1; tail -1 gpurun_out/ev3_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/ev3_bench.log 2>&1; tail -1 gpurun_out/ev3_bench.log
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/ev3_bench_$c.log 2>&1; tail -1 gpurun_out/ev3_bench_$c.log; done
bash scripts/gpu_launches.sh c5 100001 ev3_launches_c5
bash scripts/gpu_launches.sh c4 10001 ev3_launches_c4
CFG=c5 ncu --set full --clock-control none --import-source on -k regex:"ml_" -s 0 -c 6 -o gpurun_out/ev3_full_c5 -f \
    python scripts/profile_c2.py 100001 > gpurun_out/ev3_ncu_c5.log 2>&1
tail -1 gpurun_out/ev3_ncu_c5.log
