set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/r2_sweep_c1 python tools/launch_breakdown.py 1 > gpurun_out/r2_ncu_c1full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/r2_sweep_c2 python tools/launch_breakdown.py 2 > gpurun_out/r2_ncu_c2full.log 2>&1
