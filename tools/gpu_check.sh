# full GPU test suite (no -x), smoke, default bench (C5) with recall
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench=$?; tail -5 gpurun_out/bench_C5.err; tail -c 2500 gpurun_out/bench_C5.json
