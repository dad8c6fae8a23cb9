set -x
timeout 900 python tests/checks/pbbem_solve_report.py 3 4 > gpurun_out/r2r_solve_report.txt 2>&1
