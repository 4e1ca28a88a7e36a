# subtree experiment: partition tests + C2/C3/C4 partition time by PIPNN_SUBTREE_DEPTH
timeout 900 python -m pytest tests -m gpu -q -k "partition or build" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for D in 1 2 99; do for C in C2 C3 C4; do
  PIPNN_SUBTREE_DEPTH=$D python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --recall-queries 0 > gpurun_out/sub_$C.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sub_$C.json')); print('$D', '$C', round(d['ms_per_step'],3), d['stages_ms']['ms_partition'])"
done; done
