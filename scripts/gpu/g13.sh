timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_warp" -s 0 -c 6 \
    -o gpurun_out/g13_warp python scripts/prof_run.py --batches 0 --runs 1 --no-calibrate > gpurun_out/g13_ncu.log 2>&1; echo ncu rc $?
timeout 600 python -m pytest tests/test_integration_binding.py -x -q > gpurun_out/g13_tests.log 2>&1; echo tests rc $?
