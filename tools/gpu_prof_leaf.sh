# ncu --set full of the folded uint8 leaf kernel (C2 leaves), PIPNN_DEBUG_EPI=$DBG (default 0)
set -x
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:ILb1ELb0ELi8ELb1E -s 1 -c 1 -o gpurun_out/${KOUT:-leaf} python tools/leaf_exp.py ${DBG:-0} > gpurun_out/ncu_leaf.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_leaf.log
