#!/bin/bash
# ncu --set full of one vol_kernel launch per libsem variant: tools/ncu_ab.sh TAG lib1.so lib2.so ...
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
for lib in "$@"; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib $CMD > gpurun_out/plain_${TAG}_$lib.log 2>&1 && \
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib ncu --set full --clock-control none --import-source on -k regex:vol_kernel -s 4 -c 1 \
     -o gpurun_out/ncu_${TAG}_${lib%.so} $CMD > gpurun_out/ncu_${TAG}_$lib.log 2>&1
  echo "$lib rc=$?" >> gpurun_out/ncu_${TAG}.rc
done
