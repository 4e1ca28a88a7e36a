# threshold-pass tiles of the folded uint8 leaf kernel (PIPNN_P1) on C5, then an ncu source capture of it on C2
set -x
for P in 6 3 4 8 6; do
  PIPNN_P1=$P timeout 300 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-int8-peak --recall-queries 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[P1=$P]', round(d['ms_per_step'],3), d['stages_ms']['ms_leaf_tiles'])"
done
CFG=C2 KREGEX=dist_topk_uf2_kernel bash tools/gpu_prof_leaf_c5.sh
python tools/sass_hot.py gpurun_out/leaf_C2_sass.csv 40 > gpurun_out/uf2_C2_hot.txt
python tools/ncu_raw_summary.py gpurun_out/leaf_C2_raw.csv > gpurun_out/uf2_C2_ncu_summary.txt
rm -f gpurun_out/*.ncu-rep
