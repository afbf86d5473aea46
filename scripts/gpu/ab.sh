# A/B device time of library builds: bash scripts/gpu/ab.sh OUT lib1 lib2 ... (configs via $CONFIGS)
O=$1; shift; : > $O
for rep in 1 2; do
for lib in "$@"; do
  for c in ${CONFIGS:-rmat22}; do
    LP_LIB_PATH=$lib python scripts/ab_time.py --config $c --tag "$lib" >> $O 2>&1
  done
done
done
