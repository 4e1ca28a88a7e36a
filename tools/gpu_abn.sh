# A/B/n of environment settings on the C2 (or $CFG) bench: VARS="A=1 B=2|C=3" ('|'-separated, '-' = none)
IFS='|' read -ra VS <<< "${VARS}"
for r in 1 2; do
  for v in - "${VS[@]}"; do
    [ "$v" = "-" ] && v=""
    env $v timeout 300 python bench.py --config ${CFG:-C2} --steps 5 --warmup 3 --no-cpu-baseline --recall-queries 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[${v:-base}]', round(d['ms_per_step'],3), d['stages_ms'])"
  done
done
