# the partition's packed pass on dist_topk_uf2_kernel: partition/build parity, then A/B (PIPNN_UF2=1: leaves only)
set -x
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_fullsize.py tests/test_gpu_build.py tests/test_gpu_sharded.py -m gpu -x -q --timeout 600 > gpurun_out/pk_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pk_pytest.log
CFG=C5 AB=PIPNN_UF2=1 bash tools/gpu_ab.sh
CFG=C2 AB=PIPNN_UF2=1 bash tools/gpu_ab.sh
