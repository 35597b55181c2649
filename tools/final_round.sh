# Round-end validation on the GPU box: tests, smoke, the default bench line,
# the reference arm and the cfg3 launch list (run from the repo root).
set -u
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${R}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/${R}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${R}_smoke.log
timeout 600 python bench.py > gpurun_out/${R}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${R}_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${R}_bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --e2e-steps 0 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/${R}_ncu_launch.log 2>&1
echo "launch list rc=$?"; python tools/launch_summary.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches.txt; head -8 gpurun_out/${R}_launches.txt
