set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_v7.json 2> gpurun_out/bench_v7.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-2h --no-fp32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5_256_v7.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-2h --no-fp32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wc_stage -s 4 -c 1 -o gpurun_out/prof_c5_256_v7 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-2h --no-fp32 > /dev/null 2>&1
echo done
