#!/bin/bash
# C5 headline: bench line, then the ncu launch list and one --set full
# capture of a stage launch (each after the same command exited 0 without
# ncu).  Outputs in gpurun_out/:
#   gpurun --timeout 2400 -- bash scripts/profile_c5.sh
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err
python scripts/c4_profile.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tl|k_set_dt|k_speed" --csv --log-file gpurun_out/c4_launches_v4.csv python scripts/c4_profile.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tl_pass_[ab]" -s 2 -c 2 -o gpurun_out/c4_passes_v4 python scripts/c4_profile.py > /dev/null 2>&1
echo done
