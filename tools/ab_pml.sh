#!/bin/bash
# PML element-kernel A/B: GPU parity of the PML tests with the main library, then tools/ab_run.sh on
# cfg 3 + a 2-element PML for the given variant libraries, then ncu of the element kernel per library
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests -m gpu -x -q -k "pml" > gpurun_out/t_pml.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/t_pml.log
rm -f gpurun_out/ab.log
AB_ARGS="--pml 2" bash tools/ab_run.sh "$@"
for lib in "$@"; do
  SEM_LIB=$PWD/paper_2603_06267_b200/lib/$lib timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"pml_element" -s 4 -c 1 -o gpurun_out/ncu_pml_${lib%.so} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --pml 2 \
    > gpurun_out/ncu_pml_${lib%.so}.log 2>&1
done
