#!/bin/bash
# usage: tools/swap_time.sh <alt .so> ... : time the fused cfg3 call with each library variant
L=paper_2305_13925_b200/_native/libxlmimo_b200.so
cp $L /tmp/orig.so
for f in "$@"; do cp $f $L; echo "$f: $(timeout 120 python tools/time_fused.py 2>&1 | tail -1)"; done
cp /tmp/orig.so $L
