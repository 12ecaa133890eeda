#!/bin/bash
# 4 x 32 default: launch list + trace, then ncu --set full of the gather and the hop-2 sampling kernels.
bash profiles/r02_c4_list.sh r02n32; echo list=$?
bash profiles/r02_ncu_full.sh r02n32 gather_tma_kernel:8 k_tiny:26 k_compact_emit:26 k_compact_count:26 k_scatter:26 k_count:26 k_select:26
