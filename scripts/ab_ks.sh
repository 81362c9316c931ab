# A/B device times of variant libraries on config-2 windows: bash scripts/ab_ks.sh "KS" variant...
KS=$1; shift
python scripts/time_ks.py $KS
for v in "$@"; do MF_B200_LIB=$PWD/_variants/$v/libmedfilt_b200.so python scripts/time_ks.py $KS; done
python scripts/time_ks.py $KS
