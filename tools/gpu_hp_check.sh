# HashPrune iteration: hashprune/build parity, then C5 and C2 stage times
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_build.py tests/test_gpu_sharded.py -q -x --timeout 600 -k "hashprune or build" 2>&1 | tail -3
for C in ${CFGS:-C5 C2}; do
timeout 600 python bench.py --config $C --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --recall-queries 0 --no-int8-peak > gpurun_out/b_$C.json 2>gpurun_out/b_$C.err
python -c "
import json; d=json.loads(open('gpurun_out/b_$C.json').read().strip().splitlines()[-1]); print('$C', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['value']/1e6,1))" || tail -3 gpurun_out/b_$C.err
done
