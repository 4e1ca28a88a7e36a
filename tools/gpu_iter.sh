# iteration: build/stage parity tests, then C2 and C5 stage times (PYTEST_FILES / CFGS override)
timeout 900 python -m pytest ${PYTEST_FILES:-tests/test_gpu_build.py tests/test_gpu_stages.py} -q -x --timeout 600 2>&1 | tail -3
for C in ${CFGS:-C2 C5}; do
env $V timeout 600 python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --recall-queries 0 --no-int8-peak > gpurun_out/b_$C.json 2>gpurun_out/b_$C.err
python -c "
import json; d=json.loads(open('gpurun_out/b_$C.json').read().strip().splitlines()[-1]); print('[$V] $C', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/b_$C.err
done
