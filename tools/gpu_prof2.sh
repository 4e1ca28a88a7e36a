# ncu --set full captures of the leaf distance kernel and the final-prune tier-32 kernel (C2 bench workload)
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_kernelILb1ELb0ELi8E -s 1 -c 1 -o gpurun_out/prof_leaf $CMD > gpurun_out/ncu_leaf.log 2>&1; echo ncu_leaf=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:fp_gram_kernelILb1ELb0ELi32E -s 1 -c 1 -o gpurun_out/prof_fp $CMD > gpurun_out/ncu_fp.log 2>&1; echo ncu_fp=$?
tail -2 gpurun_out/ncu_leaf.log gpurun_out/ncu_fp.log
