#!/bin/bash
# C4 (TL-SPH column) ncu evidence on a GPU box; each ncu command runs only
# after the same command exited 0 without ncu (set -e).  Outputs in gpurun_out/:
#   gpurun --timeout 1200 -- bash scripts/profile_c4.sh
set -e
mkdir -p gpurun_out
python scripts/c4_profile.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tl|k_set_dt|k_speed" --csv --log-file gpurun_out/c4_launches.csv python scripts/c4_profile.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tl_zb_b|k_tl_lattice_a|k_tl_kick" -s 3 -c 3 -o gpurun_out/c4_passes python scripts/c4_profile.py > /dev/null 2>&1
echo done
