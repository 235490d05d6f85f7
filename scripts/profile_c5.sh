#!/bin/bash
# C5 headline: bench line, then the ncu launch list and one --set full
# capture of a stage launch (each after the same command exited 0 without
# ncu).  Outputs in gpurun_out/:
#   gpurun --timeout 2400 -- bash scripts/profile_c5.sh
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-2h --no-fp32 --no-c4"
$CMD > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/launches_c5_256.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_wc_(stage|lattice)' -s 4 -c 1 \
    -o gpurun_out/prof_c5_256 $CMD > /dev/null 2>&1
echo done
