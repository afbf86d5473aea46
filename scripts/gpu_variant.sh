# A/B: the default build vs a variant built with EXTRA flags (same prof runs)
# usage: bash scripts/gpu_variant.sh "-DFOO=1" [prof_run args]
VAR="$1"; shift
make -s -C paper_2301_09125_b200/csrc || exit 1
cp paper_2301_09125_b200/liblabelprop_cuda.so /tmp/lp_default.so
make -s -C paper_2301_09125_b200/csrc OUT=/tmp/lp_variant.so EXTRA="$VAR" || exit 1
for v in default variant; do
  cp /tmp/lp_$v.so paper_2301_09125_b200/liblabelprop_cuda.so
  echo "== $v exact";  python scripts/prof_run.py --no-calibrate --runs 2 "$@" 2>&1 | tail -1
  echo "== $v sync";   python scripts/prof_run.py --no-calibrate --runs 2 --batches 1 "$@" 2>&1 | tail -1
done
cp /tmp/lp_default.so paper_2301_09125_b200/liblabelprop_cuda.so
