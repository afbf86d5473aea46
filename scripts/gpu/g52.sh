O=gpurun_out/g52
timeout 1200 python -m pytest tests/test_copra_gpu.py tests/test_slpa_gpu.py -x -q -m gpu > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 ${O}_pytest.log
timeout 1200 python scripts/bench_mlp.py > ${O}_copra_slpa.jsonl 2> ${O}_copra_slpa.err
python - <<'PY'
import json
for l in open('gpurun_out/g52_copra_slpa.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    c=d.get('config',{})
    print(d['algo'], c.get('max_labels',c.get('memory_size')), 'B',c.get('batches'), 'ms',round(d['ms_per_run'],2),'gteps',round(d['value'],2),'it',d['iterations'], 'same', d.get('cpu',{}).get('same_result'))
PY
