O=gpurun_out/final
timeout 2400 python -m pytest tests -x -q -m gpu > ${O}_pytest_all.log 2>&1; echo "pytest all rc=$?"; tail -3 ${O}_pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 ${O}_smoke.log
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/final_bench.json'))
print("value",d['value'],"ms",d['ms_per_step'],"e2e",d['e2e']['value'],d['e2e']['ms_per_step'],"parity",d['parity']['labels_equal_oracle'],"launches",d['gpu_launches'], d['clocks'])
print({k:(round(v['ms_per_run'],2),v['parity']['labels_equal_oracle']) for k,v in d['configs'].items()})
PY
