#!/bin/bash
for lib in "$@"; do
SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],2), round(d['roofline']['frac'],3))"
done
