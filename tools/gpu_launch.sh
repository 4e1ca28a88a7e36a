# GPU tests (subset via PYTEST_K) + C2 bench + launch list (no --set full)
set -x
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --config ${CFG:-C2} --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 python bench.py --config ${CFG:-C2} --steps 5 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/launch_summary.py gpurun_out/launches.csv | head -30
