set -x
timeout 900 python -m pytest tests/test_gpu_singular.py -q > gpurun_out/r2g_singular.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:singular_fast -s 2 -c 1 -o gpurun_out/r2g_singular_c4 python tools/launch_breakdown.py 4 > gpurun_out/r2g_ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2g_gputest.txt 2>&1; echo "gputest rc=$?" >> gpurun_out/r2g_gputest.txt
timeout 600 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
