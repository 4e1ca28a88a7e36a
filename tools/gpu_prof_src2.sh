for K in ${KERNELS:-fp_band_kernel hp_merge_rows_kernel hp_emit_kernelIiLi512}; do K=$K bash tools/gpu_prof_src.sh > /dev/null 2>&1; echo "$K done"; done
ls gpurun_out/src_*sass.csv
