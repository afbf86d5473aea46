make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
timeout 900 python -m pytest tests/test_rak_gpu.py tests/test_slpa_gpu.py tests/test_copra_gpu.py -x -q 2>&1 | tail -3
for M in 0 1; do echo "MARGIN=$M"; LP_MARGIN=$M timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 2>&1 | tail -1; done
for M in 0 1; do echo "MARGIN=$M nonstrict"; LP_MARGIN=$M timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 --non-strict 2>&1 | tail -1; done
echo "planted"; LP_MARGIN=1 timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 --config planted 2>&1 | tail -1
echo "grid"; LP_MARGIN=1 timeout 300 python scripts/prof_run.py --no-calibrate --runs 2 --config grid 2>&1 | tail -1
for M in 0 1; do echo "slpa M=$M"; LP_MARGIN=$M python scripts/prof_mlp.py slpa 20 0 | tail -1; done
