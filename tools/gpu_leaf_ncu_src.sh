# leaf kernel A/B (tau step on/off) on C5 leaves, then an ncu source-level capture of the C2 leaf kernel
bash tools/gpu_tau_prof.sh
for V in "" PIPNN_NO_TAU=1; do
  T=$([ -z "$V" ] && echo tau || echo notau)
  env $V CFG=C2 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:ILb1ELb0ELi8ELb1E -s 1 -c 1 -o gpurun_out/leaf_$T python tools/leaf_exp.py 0 > gpurun_out/ncu_leaf_$T.log 2>&1; echo ncu=$?
  ncu -i gpurun_out/leaf_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/leaf_${T}_sass.csv 2>/dev/null
  ncu -i gpurun_out/leaf_$T.ncu-rep --page raw --csv > gpurun_out/leaf_${T}_raw.csv 2>/dev/null
done
