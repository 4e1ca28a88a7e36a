# launch list of one C5 build + ncu --set full of the HashPrune kernels
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python tools/build_once.py C5 > /dev/null 2>&1; echo launch=$?
python tools/launch_summary.py gpurun_out/launches_C5.csv | head -40
KERNELS="${KERNELS:-hp_emit_kernel hp_merge_rows_kernel hp_defer_table_kernel}" bash tools/gpu_prof_kernels.sh
for K in ${KERNELS:-hp_emit_kernel hp_merge_rows_kernel hp_defer_table_kernel}; do python tools/ncu_raw_summary.py gpurun_out/k_C5_${K}_raw.csv 2>/dev/null | head -30; done
