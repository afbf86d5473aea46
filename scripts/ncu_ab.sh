# ncu launch list (duration only) of one detection per setting: bash scripts/ncu_ab.sh "ENV=.." ...
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_l$i.csv \
      python scripts/prof_run.py --runs 1 --no-calibrate --config ${CONFIG:-rmat22} > gpurun_out/ab_l$i.log 2>&1
  echo "== $cfg" >> gpurun_out/ab_ncu.txt
  python scripts/launch_seq.py gpurun_out/ab_l$i.csv >> gpurun_out/ab_ncu.txt
  i=$((i+1))
done
cat gpurun_out/ab_ncu.txt
