#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#  1. the default bench line without a profiler,
#  2. the launch list of the same command (gpu__time_duration, serialised),
#  3. one `ncu --set full` capture of the fused kernel at batch 4096.
set -u
R=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench.log 2>&1 || { echo "bench failed"; tail -n 20 gpurun_out/${R}_bench.log; exit 1; }
tail -n 1 gpurun_out/${R}_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py > gpurun_out/${R}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python bench.py --batch 4096 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${R}_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_rzf -s 3 -c 1 -o gpurun_out/${R}_fused \
    python bench.py --batch 4096 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${R}_ncu_full.log 2>&1
echo "full capture rc=$?"
