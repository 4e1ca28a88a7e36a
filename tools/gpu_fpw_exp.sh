for V in 0 1; do
  if [ $V = 1 ]; then export PIPNN_FP_WARP_U8=1; fi
  PIPNN_DEBUG_TIMING=1 timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0 --no-int8-peak > gpurun_out/fpw_$V.json 2>gpurun_out/fpw_$V.err
  python -c "
import json; d=json.loads(open('gpurun_out/fpw_$V.json').read().strip().splitlines()[-1]); print('V$V', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
  grep -i "tier\|final" gpurun_out/fpw_$V.err | tail -3
done
