#!/bin/bash
# Round-end evidence: the default bench line, the PML variant, the ncu launch list of the default step and
# one --set full capture of the volume kernel (each ncu pass after the same command exited 0 without ncu)
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r2}
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_prof.rc
timeout 600 python bench.py --pml 2 --no-cpu-baseline > gpurun_out/${TAG}_bench_pml2.json 2> gpurun_out/${TAG}_bench_pml2.err
echo "pml rc=$?" >> gpurun_out/${TAG}_prof.rc
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg3.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vol_kernel -s 4 -c 1 -o gpurun_out/${TAG}_vol $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1 && \
ncu -i gpurun_out/${TAG}_vol.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
echo "ncu rc=$?" >> gpurun_out/${TAG}_prof.rc
