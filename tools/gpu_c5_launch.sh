# C5 launch list of one build (build_once) + per-kernel summary; optional ncu --set full of $KERNELS
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python tools/build_once.py C5 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/launch_summary.py gpurun_out/launches_C5.csv | head -40
if [ -n "$KERNELS" ]; then
  KERNELS="$KERNELS" bash tools/gpu_prof_kernels.sh
  for K in $KERNELS; do python tools/ncu_raw_summary.py gpurun_out/k_C5_${K}_raw.csv; done
fi
