# rows straight from X vs tiled leaf operands: parity, then C5 leaf-pick time / wait profile / epilogue-free floor
timeout 600 python -m pytest tests/test_gpu_leaf_pick.py tests/test_gpu_build.py -q -x --timeout 300 2>&1 | tail -3
export CFG=${CFG:-C5}
for TG in ${TGS:-1 0}; do
  for D in ${DBGS:-0 64 1}; do
    echo "== TG=$TG dbg=$D"
    PIPNN_LEAF_TG=$TG PIPNN_DEBUG_EPI=$D timeout 600 python tools/leaf_exp.py 2>&1 | tail -3
  done
done
