#!/bin/bash
# ncu --set full of the non-volume kernels of a cfg-3 + PML step (fused interface, modal, PML element and
# fix-up) and of the curved-box kernels, after plain runs of the same commands exited 0
cd ${GRAFT_REPO_ROOT:-.}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --pml 2"
timeout 300 $CMD > gpurun_out/plain_aux.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"iface_fused|modal_kernel|pml_element_kernel|pml_fixup_kernel" -s 8 -c 4 \
   -o gpurun_out/ncu_aux $CMD > gpurun_out/ncu_aux.log 2>&1
echo "aux rc=$?" >> gpurun_out/prof_aux.rc
CMD2="python tools/curved_bench.py"
timeout 300 $CMD2 > gpurun_out/plain_curved.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"curved_residual|curved_update" -s 4 -c 2 \
   -o gpurun_out/ncu_curved $CMD2 > gpurun_out/ncu_curved.log 2>&1
echo "curved rc=$?" >> gpurun_out/prof_aux.rc
