# ncu --set full of one leaf distance-tile launch (dist_topk_kernel<1,0,8>) in a C5 build + source counters
set -x
CFG=${CFG:-C5}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:${KREGEX:-dist_topk_kernelILb1ELb0ELi8E} -s 0 -c 1 -o gpurun_out/leaf_${CFG} python tools/build_once.py $CFG > gpurun_out/ncu_leaf_${CFG}.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_leaf_${CFG}.log
ncu -i gpurun_out/leaf_${CFG}.ncu-rep --page source --csv --print-source sass > gpurun_out/leaf_${CFG}_sass.csv 2>/dev/null; echo src=$?
ncu -i gpurun_out/leaf_${CFG}.ncu-rep --page raw --csv > gpurun_out/leaf_${CFG}_raw.csv 2>/dev/null; echo raw=$?
ls -la gpurun_out/leaf_${CFG}*
