# tau-step iteration: leaf-pick + build parity, then C2/C5 stage times with and without the tau step
timeout 600 python -m pytest tests/test_gpu_leaf_pick.py tests/test_gpu_build.py tests/test_gpu_quant.py -q -x --timeout 300 2>&1 | tail -3
for V in "" PIPNN_NO_TAU=1; do
for C in ${CFGS:-C2 C5}; do
env $V timeout 600 python bench.py --config $C --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --recall-queries 0 --no-int8-peak > gpurun_out/b_$C.json 2>gpurun_out/b_$C.err
python -c "
import json; d=json.loads(open('gpurun_out/b_$C.json').read().strip().splitlines()[-1]); print('[$V] $C', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/b_$C.err
done; done
