#!/bin/bash
# ncu --set full of one pair-symmetric C5 stage launch (k_wc_lattice_sym),
# after the same command exited 0 without ncu.  Outputs in gpurun_out/.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-2h --no-fp32 --no-c4 ${BENCH_ARGS}"
$CMD > gpurun_out/sym_cmd.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_wc_lattice_sym}" -s 2 -c 1 \
    -o gpurun_out/prof_sym${TAG} $CMD > gpurun_out/sym_ncu.log 2>&1
echo done
