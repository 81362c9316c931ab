# A/B timing of experiment builds: bash scripts/ab.sh "K ..." lib1.so lib2.so ...
ks="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do MF_B200_LIB=$lib python scripts/time_ks.py $ks; done
done
