set -x
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b_rmat22_exact.json 2> gpurun_out/b_rmat22_exact.err; tail -3 gpurun_out/b_rmat22_exact.err
timeout 600 python bench.py --steps 5 --warmup 3 --batches 1 --no-cpu-baseline --no-e2e > gpurun_out/b_rmat22_sync.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --batches 64 --no-cpu-baseline --no-e2e > gpurun_out/b_rmat22_b64.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --non-strict --no-cpu-baseline --no-e2e > gpurun_out/b_rmat22_ns.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --config planted --no-e2e > gpurun_out/b_planted.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --config grid --no-cpu-baseline --no-e2e > gpurun_out/b_grid.json 2>&1
cat gpurun_out/b_*.json | cut -c1-600
