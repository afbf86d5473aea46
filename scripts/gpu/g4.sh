# k_warp path statistics (LP_PATH_STATS build) + ncu --set full of the first dense round's kernels (synchronous schedule)
for b in 1 0; do LP_LIB_PATH=build/liblp_stats.so timeout 300 python scripts/prof_run.py --batches $b --runs 2 --no-calibrate > gpurun_out/g4_stats_b$b.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_warp|k_team|k_midh|k_small|k_gather_dense" -s 0 -c 10 \
    -o gpurun_out/g4_full python scripts/prof_run.py --batches 1 --runs 1 --no-calibrate > gpurun_out/g4_ncu.log 2>&1; echo ncu rc $?
