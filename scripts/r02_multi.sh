# round-2: multi-device / multi-stream tests, the full GPU suite, a bench line with checksums
set -x
python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02_multi_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_multi_pytest.log
python -m pytest tests -m gpu -x -q > gpurun_out/r02_multi_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02_multi_all.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_multi_bench.log 2>&1
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_multi_ref.log 2>&1
tail -2 gpurun_out/r02_multi_pytest.log
