# launch list of one build of config $CFG
set -x
CMD="python bench.py --config ${CFG} --steps 1 --warmup 1 --no-cpu-baseline --recall-queries 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${CFG}.csv $CMD > gpurun_out/ncu_launch_${CFG}.log 2>&1; echo ncu_launch=$?
