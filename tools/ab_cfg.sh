#!/bin/bash
# usage: tools/ab_cfg.sh <variant> ... : interleaved cfg2 / cfg3 timing of variants/<variant>.so
L=paper_2305_13925_b200/_native/libxlmimo_b200.so
cp $L /tmp/orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp variants/$v.so $L
    echo "$v cfg2: $(python tools/time_fused.py cfg2 65536 2>&1 | tail -1)   cfg3: $(python tools/time_fused.py cfg3 32768 2>&1 | tail -1)"
  done
done
cp /tmp/orig.so $L
