#!/bin/bash
# usage: tools/swap_bench.sh <alt .so> ... : bench each library variant in turn
L=paper_2305_13925_b200/_native/libxlmimo_b200.so
cp $L /tmp/orig.so
for f in "$@"; do cp $f $L; echo "$f: $(timeout 120 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-110)"; done
cp /tmp/orig.so $L
