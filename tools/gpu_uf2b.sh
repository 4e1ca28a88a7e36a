set -x
timeout 900 python -m pytest tests/test_gpu_leaf_pick.py tests/test_gpu_build.py -m gpu -x -q --timeout 300 > gpurun_out/uf2_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/uf2_pytest.log
for P in 6 3 4 6 3 4; do
  PIPNN_P1=$P timeout 300 python bench.py --config ${CFG:-C5} --steps 3 --warmup 3 --no-cpu-baseline --no-int8-peak --recall-queries 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[P1=$P]', round(d['ms_per_step'],3), d['stages_ms']['ms_leaf_tiles'])"
done
