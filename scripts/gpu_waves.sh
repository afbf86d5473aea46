make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_slpa_gpu.py -x -q 2>&1 | tail -3
for W in 1 4 8 16 32; do echo "W=$W"; LP_WAVES=$W timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 2>&1 | tail -1; done
for W in 1 8 16; do echo "slpa W=$W"; LP_WAVES=$W python scripts/prof_mlp.py slpa 20 0 | tail -1; done
