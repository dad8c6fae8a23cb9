set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 3 -o gpurun_out/r2_sweep_b python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/r2_ncu_full_b.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tall4.log 2>&1
