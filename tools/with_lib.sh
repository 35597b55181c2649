#!/bin/bash
# usage: tools/with_lib.sh <variant.so> <command...>
# Run a command with a variant library (e.g. the development-hooks build:
#   python paper_2305_13925_b200/build_ext.py --out variants/dev.so -DXL_DEV_HOOKS=1)
# swapped in for the in-tree libxlmimo_b200.so, restoring it afterwards.
L=paper_2305_13925_b200/_native/libxlmimo_b200.so
so=$1; shift
cp $L /tmp/with_lib_orig.so
cp "$so" $L
"$@"; rc=$?
cp /tmp/with_lib_orig.so $L
exit $rc
