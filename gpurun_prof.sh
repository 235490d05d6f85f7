set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_v8.json 2> gpurun_out/bench_v8.err
python scripts/c4_profile.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tl|k_set_dt|k_speed" --csv --log-file gpurun_out/c4_launches_v4.csv python scripts/c4_profile.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tl_pass_[ab]" -s 2 -c 2 -o gpurun_out/c4_passes_v4 python scripts/c4_profile.py > /dev/null 2>&1
echo done
