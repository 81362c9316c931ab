set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_run2_all.log 2>&1; echo "rc=$?" >> gpurun_out/r02_run2_all.log
bash scripts/r02_sanitize.sh
