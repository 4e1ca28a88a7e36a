set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --recall-queries 0"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dist_topk -s 6 -c 1 -o gpurun_out/prof_leaf2 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$?; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
