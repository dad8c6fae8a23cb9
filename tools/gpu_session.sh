set -x
timeout 1200 python -m pytest tests/test_gpu_scale_golden.py -q > gpurun_out/r2t_scale.txt 2>&1; echo "rc=$?" >> gpurun_out/r2t_scale.txt
