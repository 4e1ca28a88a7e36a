# per-launch durations of the final-prune kernels in one C5 build, for library variants gpurun_var/lib_$V.so
for V in ${VARS:-head pipe}; do
  cp gpurun_var/lib_$V.so paper_2602_21247_b200/libpipnn.so
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KRE:-fp_}" --csv python tools/build_once.py ${CFG:-C5} 2>/dev/null | grep -v "^==" > gpurun_out/fpcmp_$V.csv
  echo "== $V"; python - $V <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/fpcmp_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    print(r[h.index("Kernel Name")][:40], r[h.index("Metric Value")])
PY
done
