# quick GPU check: parity tests + bench (no ncu)
set -x
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --recall-queries ${RQ:-300} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
