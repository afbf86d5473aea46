mkdir -p gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-modes --no-kernel-events > gpurun_out/m_noev.json 2> gpurun_out/m_noev.err
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-modes > gpurun_out/m_ev.json 2> gpurun_out/m_ev.err
python -c "
import json
for f in ('m_noev','m_ev'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['value'], d['ms_per_step'])"
