# profile: launch list + ncu --set full of the kernel matching $KREGEX (skip $KSKIP launches)
set -x
CMD="python bench.py --config ${CFG:-C2} --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${KSKIP:-0} -c ${KCOUNT:-1} -o gpurun_out/${KOUT:-prof} $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
tail -3 gpurun_out/ncu_full.log
