set -x
timeout 1500 python tools/size_sweep.py > gpurun_out/r2u_size_sweep.md 2> gpurun_out/r2u_size_sweep.err
timeout 900 python tools/solve_table.py 1 2 3 4 > gpurun_out/r2u_solve_table.jsonl 2> gpurun_out/r2u_solve_table.err
