O=gpurun_out/g57
timeout 2400 python -m pytest tests -x -q -m gpu > ${O}_pytest_all.log 2>&1; echo "pytest all rc=$?"; tail -3 ${O}_pytest_all.log
timeout 600 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 ${O}_smoke.log
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/g57_bench.json'))
print("value",d['value'],"ms",d['ms_per_step'],"e2e",d['e2e']['value'],d['e2e']['ms_per_step'],"parity",d['parity']['labels_equal_oracle'],"launches",d['gpu_launches'])
PY
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_ref.json 2> ${O}_ref.err; echo "ref rc=$?"; head -c 400 ${O}_ref.json
