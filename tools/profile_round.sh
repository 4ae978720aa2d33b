# bench line, launch list of one bench step, and one --set full capture of the RPY kernel
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rpy_sym_kernel -s 3 -c 1 -o gpurun_out/rpy_sym_final \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
python tools/rpy6_time.py > gpurun_out/rpy6_time.txt 2>&1
