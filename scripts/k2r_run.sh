#!/bin/bash
# K2 resident-form iteration on the GPU box (dev aid): phase trace (probe build) per thread count and
# SiLU on/off, then the normal build's form timings per thread count.
set -u
M="make -C paper_2407_02031_b200/csrc -j16"
F="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
$M clean > /dev/null; $M NVFLAGS="$F -DSDB_RS_TRACE" > /dev/null 2>&1
for t in ${THREADS:-512 768 1024}; do for s in 1 0; do echo "== threads $t silu $s"; SILU=$s SDB_GN_RS_THREADS=$t timeout 120 python scripts/k2r_trace.py "$@"; done; done > gpurun_out/k2r_trace.log 2>&1
$M clean > /dev/null; $M > /dev/null 2>&1
for t in ${THREADS:-512 768 1024}; do echo "== threads $t"; SDB_GN_RS_THREADS=$t timeout 240 python scripts/k2_resident.py; done > gpurun_out/k2r.log 2>&1
