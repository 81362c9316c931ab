# full ncu capture of selected kernels: bash scripts/gpu_prof1.sh "<ks>" <regex> <count> <name>
python scripts/profile_c2.py $1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c $3 -o gpurun_out/$4 -f \
    python scripts/profile_c2.py $1 > gpurun_out/ncu_$4.log 2>&1
tail -2 gpurun_out/ncu_$4.log
