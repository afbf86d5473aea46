make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_copra_gpu.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests/test_slpa_gpu.py -x -q 2>&1 | tail -5
