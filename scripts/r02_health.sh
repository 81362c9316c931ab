timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_health_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_health_pytest.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/ev_bench_c5.log 2>&1
timeout 300 python bench.py > gpurun_out/r02_health_bench.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_health_pytest.log 2>&1
tail -3 gpurun_out/r02_health_pytest.log; tail -1 gpurun_out/r02_health_bench.log | cut -c1-300
