# full gpu tests (incl. float-weight determinism) + bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g9_tests.log 2>&1; echo tests rc $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err; echo bench rc $?
