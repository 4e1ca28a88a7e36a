# mid-round evidence: GPU tests, smoke, the default bench (C5), C2 line, C5 launch list, ncu --set full of the C5 leaf kernel
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench=$?; tail -c 600 gpurun_out/ev_bench.json
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-int8-peak > gpurun_out/ev_bench_C2.json 2> gpurun_out/ev_bench_C2.err; echo bench_C2=$?
CMD="python tools/build_once.py C5"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_C5.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_uf2_kernelILi8ELb0E -s 2 -c 1 -o gpurun_out/ev_leaf_C5 $CMD > gpurun_out/ev_ncu_leaf.log 2>&1; echo ncu_leaf=$?
ncu -i gpurun_out/ev_leaf_C5.ncu-rep --page raw --csv > gpurun_out/ev_leaf_C5_raw.csv 2>/dev/null
python tools/ncu_raw_summary.py gpurun_out/ev_leaf_C5_raw.csv > gpurun_out/ev_leaf_C5_ncu_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
