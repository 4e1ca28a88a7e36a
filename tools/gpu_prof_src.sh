# ncu --set full with source correlation for one kernel ($K) of one build of $CFG: sass and cuda source pages
CFG=${CFG:-C5}
K=${K:-fp_gram_kernel}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$K -s ${SKIP:-0} -c 1 -o gpurun_out/src_$K python tools/build_once.py $CFG > gpurun_out/src_$K.log 2>&1; echo ncu=$?
ncu -i gpurun_out/src_$K.ncu-rep --page raw --csv > gpurun_out/src_${K}_raw.csv 2>/dev/null
ncu -i gpurun_out/src_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${K}_sass.csv 2>/dev/null
ncu -i gpurun_out/src_$K.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${K}_cuda.csv 2>/dev/null
rm -f gpurun_out/src_$K.ncu-rep
ls -la gpurun_out/src_${K}*
