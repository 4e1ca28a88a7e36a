for V in "" PIPNN_NO_TAU=1; do
  echo "[$V]"; env $V PIPNN_DEBUG_EPI=64 CFG=${CFG:-C5} timeout 900 python tools/leaf_exp.py 64 2>&1 | tail -4
  env $V CFG=${CFG:-C5} timeout 900 python tools/leaf_exp.py 0 2>&1 | tail -1
done
