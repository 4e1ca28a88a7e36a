# round evidence: GPU tests, smoke, the default bench (C5, full), the reference arm, other configs, the C5 launch
# list, ncu --set full captures of the C5 leaf kernel and of the HashPrune / final-prune kernels
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench=$?; tail -c 1500 gpurun_out/ev_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo ref=$?
for C in ${CFGS:-C2 C3 C4 C1 C2-f10x3 C2-rep2}; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-int8-peak > gpurun_out/ev_bench_$C.json 2> gpurun_out/ev_bench_$C.err; echo bench_$C=$?; done
timeout 300 python bench.py --config C2 --shard --steps 3 --warmup 2 > gpurun_out/ev_bench_C2-shard1.json 2> gpurun_out/ev_bench_shard.err; echo shard=$?
timeout 300 python bench.py --config C3 --quant --steps 5 --warmup 3 --no-cpu-baseline --no-int8-peak --recall-queries 2000 > gpurun_out/ev_bench_C3-quant.json 2> gpurun_out/ev_bench_quant.err; echo quant=$?
CMD="python tools/build_once.py C5"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_C5.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_uf2_kernelILi8ELb0E -s 2 -c 1 -o gpurun_out/ev_leaf_C5 $CMD > gpurun_out/ev_ncu_leaf.log 2>&1; echo ncu_leaf=$?
ncu -i gpurun_out/ev_leaf_C5.ncu-rep --page raw --csv > gpurun_out/ev_leaf_C5_raw.csv 2>/dev/null
KERNELS="hp_emit_kernel hp_merge_rows_kernel hp_defer_sort_kernel fp_gram_kernel fp_band_kernel dist_topk_uf2_kernelILi2ELb1E leaders_kernel" bash tools/gpu_prof_kernels.sh
for K in hp_emit_kernel hp_merge_rows_kernel hp_defer_sort_kernel fp_gram_kernel fp_band_kernel dist_topk_uf2_kernelILi2ELb1E leaders_kernel; do
  echo "== $K"; python tools/ncu_raw_summary.py gpurun_out/k_C5_${K}_raw.csv
done > gpurun_out/ev_kernels_C5_ncu_summary.txt 2>&1
python tools/ncu_raw_summary.py gpurun_out/ev_leaf_C5_raw.csv > gpurun_out/ev_leaf_C5_ncu_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/k_C5_*_sass.csv
