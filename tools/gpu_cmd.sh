# one gpurun call: GPU tests, bench, launch list, ncu --set full of the leaf kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dist_topk -s 8 -c 1 -o gpurun_out/prof_leaf $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
