# ncu --set full of one launch each of the named kernels in one build of $CFG (default C5); raw csv summaries
CFG=${CFG:-C5}
for K in ${KERNELS:-fp_gram_kernel hp_merge_inst_kernel hp_emit_kernel fp_band_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s 0 -c 1 -o gpurun_out/k_${CFG}_$K python tools/build_once.py $CFG > /dev/null 2>&1
  ncu -i gpurun_out/k_${CFG}_$K.ncu-rep --page raw --csv > gpurun_out/k_${CFG}_${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/k_${CFG}_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/k_${CFG}_${K}_sass.csv 2>/dev/null
  echo "$K done"
done
