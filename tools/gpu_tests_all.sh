# all GPU tests, no -x (full failure pattern), then bench
set -x
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -30
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --recall-queries ${RQ:-300} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
