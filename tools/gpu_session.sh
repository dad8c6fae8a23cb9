set -x
timeout 900 python -m pytest tests/test_gpu_gmres_graph.py tests/test_hypot.py -x -q -p no:cacheprovider > gpurun_out/r2_t4.log 2>&1
timeout 300 python tools/solve_table.py 1 2 3 4 > gpurun_out/r2_solve_table3.jsonl 2>&1
HOBI_GMRES_GRAPH=0 timeout 300 python tools/solve_table.py 1 2 3 4 > gpurun_out/r2_solve_table3_nograph.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tall3.log 2>&1
