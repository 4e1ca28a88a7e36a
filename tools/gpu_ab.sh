# A/B of an environment switch on the C2 (or $CFG) bench: stage times, 2 alternating runs each
for r in 1 2; do
  for v in "" "$AB"; do
    env $v timeout 300 python bench.py --config ${CFG:-C2} --steps 5 --warmup 3 --no-cpu-baseline --recall-queries 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[${v:-base}]', round(d['ms_per_step'],3), d['stages_ms'])"
  done
done
