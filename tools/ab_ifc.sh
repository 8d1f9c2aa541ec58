#!/bin/bash
# interface-kernel A/B on cfg 3: the profiling pass's interface ms/step per libsem variant
cd ${GRAFT_REPO_ROOT:-.}
for lib in "$@"; do
SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', round(d['value'],2), round(r['frac'],3), 'iface', round(r['interface_ms_per_step'],4), 'modal', round(r['modal_ms_per_step'],4), [round(x,1) for x in d['repeats_ms']])" >> gpurun_out/ab_ifc.log
done
