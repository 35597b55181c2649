set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cluster_pcg.py -x -q > gpurun_out/cp_tests.log 2>&1; echo "cluster tests rc=$?"; tail -25 gpurun_out/cp_tests.log
for s in cluster gemm; do
  if [ $s = gemm ]; then export XL_LARGE_K_SOLVER=gemm; else unset XL_LARGE_K_SOLVER; fi
  timeout 300 python tools/time_fused.py cfg4 2048 2>&1 | tail -1 | sed "s/^/$s cfg4: /"
done
unset XL_LARGE_K_SOLVER
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cp_all.log 2>&1; echo "all gpu rc=$?"; tail -3 gpurun_out/cp_all.log
