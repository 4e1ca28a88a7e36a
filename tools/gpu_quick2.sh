# GPU suite (no -x), then the default bench without the slow extras, then one debug-timing build of C5
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -30
timeout 900 python bench.py --no-cpu-baseline --no-int8-peak --recall-queries ${RQ:-1000} > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench=$?; tail -3 gpurun_out/bench_C5.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_C5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages_ms'], d.get('recall_at_10'), d['e2e']['value'])"
PIPNN_DEBUG_TIMING=1 timeout 300 python tools/build_once.py C5 2>&1 | grep hashprune
