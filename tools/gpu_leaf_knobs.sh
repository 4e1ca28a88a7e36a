# leaf-pick time under debug-knob variants (each its own process: knobs are read once): DBGS="0 128 256"
export CFG=${CFG:-C5}
for D in ${DBGS:-0}; do
  echo "== dbg=$D"
  PIPNN_DEBUG_EPI=$D timeout 600 python tools/leaf_exp.py 2>&1 | tail -1
done
