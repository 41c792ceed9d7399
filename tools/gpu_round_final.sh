# One GPU round: parity suite, smoke, default bench, ncu launch list of a short bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench exit $?"
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches.csv python tools/ncu_target.py 1 2000 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1; head -8 gpurun_out/launch_summary.txt
