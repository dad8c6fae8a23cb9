set -x
timeout 1200 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_kirkwood.py -q -p no:cacheprovider > gpurun_out/r2_t3.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_b5.json 2> gpurun_out/r2_b5.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_ref5.json 2> gpurun_out/r2_ref5.err
