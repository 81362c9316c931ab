python scripts/e2e_chunks.py 4194304 8388608 2>&1 | tail -2
for v in ramp8 ramp32 slots6 slots3; do echo $v; MF_B200_LIB=$PWD/_variants/$v/libmedfilt_b200.so python scripts/e2e_chunks.py 4194304 8388608 2>&1 | tail -2; done
