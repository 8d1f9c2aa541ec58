#!/bin/bash
# A/B of libsem variants on cfg 3: tools/ab_run.sh lib1.so lib2.so ... (2 passes, bench.py graph path)
cd ${GRAFT_REPO_ROOT:-.}
for i in 1 2; do
for lib in "$@"; do
SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $AB_ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],2), round(d['roofline']['frac'],3), 'if', round(d['roofline'].get('interface_ms_per_step',0),4), 'mo', round(d['roofline'].get('modal_ms_per_step',0),4), 'pml', round(d['config'].get('pml',{}).get('element_kernel_ms_per_step',0),4), [round(x,1) for x in d['repeats_ms']], d['clocks'])" >> gpurun_out/ab.log
done; done
