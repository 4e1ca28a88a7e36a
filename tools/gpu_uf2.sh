# parity of the four-warpgroup folded-uint8 leaf kernel, then its A/B against dist_topk_kernel (PIPNN_UF2=0)
set -x
timeout 900 python -m pytest tests/test_gpu_leaf_pick.py tests/test_gpu_build.py -m gpu -x -q --timeout 300 > gpurun_out/uf2_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/uf2_pytest.log
CFG=C2 AB=PIPNN_UF2=0 bash tools/gpu_ab.sh
CFG=C5 AB=PIPNN_UF2=0 bash tools/gpu_ab.sh
