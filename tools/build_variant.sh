#!/bin/bash
# build_variant.sh NAME "-DSEM_KTY=.. -DSEM_KPREF=.. ..."  -> paper_2603_06267_b200/lib/libsem_NAME.so
set -e
cd "$(dirname "$0")/.."
C=paper_2603_06267_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC $2"
nvcc $F -Xptxas -v -c $C/kernels.cu -o /tmp/k_$1.o 2>&1 | grep -A2 "vol_kernelILi5" | grep -E "spill|regis" | tr '\n' ' '; echo
nvcc $F -c $C/sem_abi.cu -o /tmp/a_$1.o
nvcc $F -c $C/matching.cu -o /tmp/m_$1.o
nvcc -shared /tmp/k_$1.o /tmp/a_$1.o /tmp/m_$1.o -o paper_2603_06267_b200/lib/libsem_$1.so
