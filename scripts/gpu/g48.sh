O=gpurun_out/g48
timeout 900 python bench.py --steps 10 --warmup 3 > ${O}_bench.json 2> ${O}_bench.err; python - <<'PY'
import json
d=json.load(open('gpurun_out/g48_bench.json'))
print("value",d['value'],"ms",d['ms_per_step'],"e2e",d['e2e'])
PY
: > ${O}_time.log
for F in 0 1; do
LP_FUSE_FRONTIER=$F timeout 600 python scripts/ab_time.py --config rmat22 --runs 9 --batches 0 --tag "ff=$F" >> ${O}_time.log 2>&1
LP_FUSE_FRONTIER=$F timeout 600 python scripts/ab_time.py --config grid --runs 5 --batches 0 --tag "ff=$F" >> ${O}_time.log 2>&1
done
cat ${O}_time.log
