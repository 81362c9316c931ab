# round-2 baseline: GPU tests, bench, fresh ncu --set full with source of the c2 medium/small kernels
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_base_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_base_pytest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_base_bench.log 2>&1
python scripts/time_ks.py 3 31 255 1023 > gpurun_out/r02_base_ks.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mf_ -s 2 -c 6 -o gpurun_out/r02_base_c2 -f \
    python scripts/profile_c2.py 31 255 1023 > gpurun_out/r02_base_ncu.log 2>&1
tail -3 gpurun_out/r02_base_ncu.log
