#!/bin/bash
# A/B of the curved-box residual kernel: tools/ab_curved.sh lib1.so lib2.so ... (curved_bench.py, 2 passes),
# then one ncu --set full capture of curved_residual_kernel per library
cd ${GRAFT_REPO_ROOT:-.}
for i in 1 2; do
for lib in "$@"; do
  echo "$lib $(SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib timeout 300 python tools/curved_bench.py 96 96 24 5 20)" >> gpurun_out/ab_curved.log
done; done
for lib in "$@"; do
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"curved_residual" -s 4 -c 1 -o gpurun_out/ncu_cv_${lib%.so} python tools/curved_bench.py 96 96 24 5 4 \
    > gpurun_out/ncu_cv_${lib%.so}.log 2>&1
done
