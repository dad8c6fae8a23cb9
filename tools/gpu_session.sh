set -x
timeout 900 python -m pytest tests/test_gpu_scale_golden.py -q -k "not 4-lobi" > gpurun_out/r2v_scale.txt 2>&1; echo "rc=$?" >> gpurun_out/r2v_scale.txt
timeout 900 python tests/checks/pbbem_solve_report.py 3 4 3lobi > gpurun_out/r2v_solve_report.txt 2>&1
