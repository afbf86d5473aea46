# usage: bash scripts/gpu_launches.sh <tag> [prof_run args...]
tag=$1; shift
mkdir -p gpurun_out
make -s -C paper_2301_09125_b200/csrc && make -s -C oracle
python scripts/prof_run.py "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python scripts/prof_run.py "$@" > gpurun_out/ncu_$tag.log 2>&1
cat gpurun_out/plain_$tag.log
python scripts/launch_table.py gpurun_out/launches_$tag.csv
