# GPU tests + bench of C2, C3, C4 (no cpu baseline; short recall)
set -x
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -12
for C in C2 C3 C4; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --recall-queries ${RQ:-0} > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; echo bench_$C=$?; tail -2 gpurun_out/bench_$C.err; done
