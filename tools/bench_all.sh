#!/bin/bash
# Every config's bench line on one box (run from the repo root): R=<tag> bash tools/bench_all.sh
set -u
R=${R:-r02}
mkdir -p gpurun_out
for c in cfg3 cfg2 cfg1 cfg4 cfg5 cfg5_c128; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${R}_bench_$c.log 2>&1
  echo "$c rc=$? $(tail -1 gpurun_out/${R}_bench_$c.log | cut -c1-160)"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_reference.log 2>&1
echo "reference rc=$? $(tail -1 gpurun_out/${R}_bench_reference.log | cut -c1-160)"
