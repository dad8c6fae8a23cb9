set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2o_launch_list_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/r2o_ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/r2o_launch_list_c4.csv > gpurun_out/r2o_launch_summary_c4.txt 2>&1
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r2o_bench_c5.json 2> gpurun_out/r2o_bench_c5.err
