#!/bin/bash
# usage: prof_cmd.sh <tag> -- profile bench.py (cfg3): ncu launch list + one --set full capture of vol_kernel
TAG=${1:-r1}
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vol_kernel -s 3 -c 1 -o gpurun_out/vol_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "prof rc=$?"
