set -x
timeout 600 python -m pytest tests/test_gpu_p2p_ranks.py tests/test_gpu_singular.py -x -q -p no:cacheprovider > gpurun_out/r2_t2.log 2>&1
