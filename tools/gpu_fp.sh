# per-launch times of the final-prune kernels for C2, C3, C4 (ncu, kernel durations only)
for C in ${CFGS:-C2 C3 C4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_|final_prune" -c 20 --csv --log-file gpurun_out/fp_$C.csv python bench.py --config $C --steps 1 --warmup 2 --no-cpu-baseline --recall-queries 0 > /dev/null 2>&1
  echo "== $C"; python tools/launch_summary.py gpurun_out/fp_$C.csv
done
