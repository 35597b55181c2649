#!/bin/bash
# usage: bash tools/microbench/energy.sh  (on the GPU box) -> gpurun_out/energy.log
cd "$(dirname "$0")"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o energy energy.cu || exit 1
nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm --format=csv,noheader -lms 50 > ../../gpurun_out/energy_smi.csv &
SMI=$!
./energy > ../../gpurun_out/energy.log
kill $SMI
cat ../../gpurun_out/energy.log
