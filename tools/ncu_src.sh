#!/bin/bash
# ncu --set full + source-level (SASS) stall export of one vol_kernel launch per variant
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
for lib in "$@"; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib timeout 300 $CMD > gpurun_out/plain_${TAG}_$lib.log 2>&1 && \
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:vol_kernel -s 4 -c 1 \
     -o gpurun_out/ncu_${TAG}_${lib%.so} $CMD > gpurun_out/ncu_${TAG}_$lib.log 2>&1 && \
  ncu -i gpurun_out/ncu_${TAG}_${lib%.so}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_${lib%.so}.csv 2>/dev/null
  echo "$lib rc=$?" >> gpurun_out/ncu_${TAG}.rc
done
