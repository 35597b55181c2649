# Large-K (K = 128) path on the GPU: parity tests, then cfg4 timing per variant.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cluster_pcg.py -x -q > gpurun_out/cp_tests.log 2>&1; echo "large-K tests rc=$?"; tail -25 gpurun_out/cp_tests.log
for v in stream:cluster library:cluster library:gemm; do
  g=${v%%:*}; s=${v##*:}
  XL_LARGE_K_GEMM=$g XL_LARGE_K_SOLVER=$s timeout 300 python tools/time_fused.py cfg4 2048 2>&1 | tail -1 | sed "s/^/$v cfg4: /"
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/cp_all.log 2>&1; echo "all gpu rc=$?"; tail -3 gpurun_out/cp_all.log
