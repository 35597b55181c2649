#!/bin/bash
# usage: tools/ab.sh "<label>|<so>|<env>" ... : time each (library, env) pair, twice, interleaved
L=paper_2305_13925_b200/_native/libxlmimo_b200.so
cp $L /tmp/orig.so
for rep in 1 2; do
  for spec in "$@"; do
    IFS='|' read -r label so envs <<< "$spec"
    cp $so $L
    echo "$label: $(env $envs timeout 120 python tools/time_fused.py 2>&1 | tail -1)"
  done
done
cp /tmp/orig.so $L
