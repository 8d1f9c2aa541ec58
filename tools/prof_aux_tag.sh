#!/bin/bash
# ncu --set full of the non-volume kernels of a cfg-3 + PML step (fused interface, modal, PML element and
# fix-up) with source-level export of the fused interface kernel, after a plain run exited 0:
#   tools/prof_aux_tag.sh TAG
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r2}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --pml 2"
timeout 300 $CMD > gpurun_out/${TAG}_plain_aux.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"iface_fused|modal_kernel|pml_element_kernel|pml_fixup" -s 8 -c 4 \
   -o gpurun_out/${TAG}_ncu_aux $CMD > gpurun_out/${TAG}_ncu_aux.log 2>&1 && \
ncu -i gpurun_out/${TAG}_ncu_aux.ncu-rep --page source --csv --print-source sass -k regex:iface_fused > gpurun_out/${TAG}_src_iface.csv 2>/dev/null
echo "aux rc=$?" >> gpurun_out/${TAG}_prof_aux.rc
