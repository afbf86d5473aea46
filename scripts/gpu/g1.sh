set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; echo tests rc $?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench rc $?
LP_DEBUG_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-modes --no-kernel-events > gpurun_out/g1_dbg_exact.json 2> gpurun_out/g1_dbg_exact.err
LP_DEBUG_ROUNDS=1 timeout 300 python bench.py --batches 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-modes --no-kernel-events > gpurun_out/g1_dbg_sync.json 2> gpurun_out/g1_dbg_sync.err
