# leaf kernel study at C5: timings under debug knobs, wait profile, ncu source-level capture of one launch
set -x
export CFG=C5
for D in 0 64 1 65; do PIPNN_DEBUG_EPI=$D timeout 600 python tools/leaf_exp.py; done 2>&1 | grep -v Warning
for P in 1 2 4; do PIPNN_P1=$P timeout 600 python tools/leaf_exp.py; done 2>&1 | grep -v Warning
KREGEX=dist_topk_kernelILb1ELb0ELi8ELb1E bash tools/gpu_prof_leaf_c5.sh
