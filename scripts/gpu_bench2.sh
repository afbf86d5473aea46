mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python bench.py > gpurun_out/b2_default.json 2> gpurun_out/b2_default.err; tail -2 gpurun_out/b2_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b2_reference.json 2>&1
python bench.py --batches 1 --no-cpu-baseline --no-e2e > gpurun_out/b2_sync.json 2>&1
python bench.py --non-strict --no-cpu-baseline --no-e2e > gpurun_out/b2_ns.json 2>&1
python bench.py --config rmat22w --no-cpu-baseline --no-e2e > gpurun_out/b2_w.json 2>&1
python bench.py --config planted --no-e2e > gpurun_out/b2_planted.json 2>&1
python bench.py --config grid --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_grid.json 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b2_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r01.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_b2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gather_dense|k_warp" -s 4 -c 4 -o gpurun_out/prof_bench_r01 python scripts/prof_run.py > gpurun_out/ncu_b2full.log 2>&1
ls -la gpurun_out/b2_* gpurun_out/*r01*
