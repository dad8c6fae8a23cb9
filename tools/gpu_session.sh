set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tall2.log 2>&1
timeout 300 python tools/solve_table.py 1 2 > gpurun_out/r2_solve_table2.jsonl 2>&1
HOBI_GMRES_TRACE=1 timeout 300 python tools/solve_table.py 1 2 > gpurun_out/r2_gmres_trace2.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_b4.json 2> gpurun_out/r2_b4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_c1b.csv python tools/launch_breakdown.py 1 > gpurun_out/r2_ncu_c1b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 3 -o gpurun_out/r2_sweep python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/r2_ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/r2_ncu_c4.log 2>&1
