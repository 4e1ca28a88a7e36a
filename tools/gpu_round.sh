# round evidence: GPU tests, smoke, full bench (cpu_baseline + recall), reference arm, the other configs,
# launch list, ncu of the leaf kernel and of the depth-0 partition kernel
set -x
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?; cat gpurun_out/bench_full.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; cat gpurun_out/bench_ref.json
for C in C1 C3 C4 C2-f10x3 C2-rep2; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; echo bench_$C=$?; done
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench_C5=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_kernelILb1ELb0ELi8E -s 1 -c 1 -o gpurun_out/prof_leaf $CMD > gpurun_out/ncu_leaf.log 2>&1; echo ncu_leaf=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_kernelILb1ELb0ELi2E -s 0 -c 1 -o gpurun_out/prof_part python tools/build_once.py > gpurun_out/ncu_part.log 2>&1; echo ncu_part=$?
