# weighted R-MAT-22 per-round breakdown; COPRA / SLPA lines; ncu launch list of one COPRA k=8 run
LP_DEBUG_ROUNDS=1 python scripts/ab_time.py --config rmat22w --batches 0 --runs 1 > gpurun_out/g10_dbg_w.log 2>&1
python scripts/bench_mlp.py --no-cpu > gpurun_out/g10_mlp.jsonl 2> gpurun_out/g10_mlp.err
cat > /tmp/copra1.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2301_09125_b200 as lp
from paper_2301_09125_b200 import _lib
from paper_2301_09125_b200.copra import copra_run
g = lp.rmat(20, seed=1); dg = _lib.DeviceGraph(g)
for K in (8,):
    p = lp.CopraParams(max_labels=K, max_iterations=20, seed=1)
    for r in range(2):
        best, it, _, _, _, st, _ = copra_run(g, p, want_sets=False, device_graph=dg)
        print(K, it, st["kernel_ms"], st.get("rounds"), flush=True)
PY
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/g10_copra_launches.csv python /tmp/copra1.py > gpurun_out/g10_copra_ncu.log 2>&1
python /tmp/copra1.py > gpurun_out/g10_copra_plain.log 2>&1
