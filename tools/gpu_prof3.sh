# launch list + ncu --set full of: partition distance kernel (first launch = depth 0), leaf kernel, hp merge
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:dist_topk_kernelILb1ELb0ELi2E -s 0 -c 1 -o gpurun_out/prof_part $CMD > gpurun_out/ncu_part.log 2>&1; echo ncu_part=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:hp_merge_inst_kernel -s 1 -c 1 -o gpurun_out/prof_hp $CMD > gpurun_out/ncu_hp.log 2>&1; echo ncu_hp=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:hp_emit_kernel -s 1 -c 1 -o gpurun_out/prof_emit $CMD > gpurun_out/ncu_emit.log 2>&1; echo ncu_emit=$?
