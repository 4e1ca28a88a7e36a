# kernel timeline of one C5 build (CUPTI): idle gaps between kernels, per-kernel time; host timing of the partition levels
set -x
timeout 600 python tools/timeline.py C5 > gpurun_out/timeline_C5.txt 2>&1; echo tl=$?
PIPNN_DEBUG_TIMING=1 timeout 600 python tools/build_once.py C5 > gpurun_out/timing_C5.txt 2>&1; echo tm=$?
tail -60 gpurun_out/timeline_C5.txt
