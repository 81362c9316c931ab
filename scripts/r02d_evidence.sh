# round-2, fourth session evidence: bench (default + every config), reference arm, launch list, ncu of the c2 kernels
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/ev4_bench_c2.log 2>&1
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ev4_bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ev4_ref_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-check > gpurun_out/ev4_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mf_ -s 1 -c 8 -o gpurun_out/ev4_c2 -f \
    python scripts/profile_c2.py 3 31 255 1023 > gpurun_out/ev4_ncu_full.log 2>&1
tail -1 gpurun_out/ev4_ncu_full.log
python scripts/time_ks.py 3 5 7 15 23 31 33 45 53 63 101 127 255 257 511 1023 > gpurun_out/ev4_ks.log 2>&1
