# GPU suite and the sanitizer cases against the bounds-checked build (MF_CHECK=1)
export MF_B200_LIB=$PWD/_variants/check/libmedfilt_b200.so
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_checked_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02_checked_pytest.log
python scripts/sanitize_cases.py > gpurun_out/r02_checked_cases.log 2>&1; echo "rc=$?" >> gpurun_out/r02_checked_cases.log
tail -3 gpurun_out/r02_checked_pytest.log
