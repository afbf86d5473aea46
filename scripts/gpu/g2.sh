# full-size parity tests + the new bench line (both arms)
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -x -q -s > gpurun_out/g2_fullsize.log 2>&1; echo fullsize rc $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo bench rc $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g2_ref.json 2> gpurun_out/g2_ref.err; echo ref rc $?
