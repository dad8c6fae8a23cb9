set -x
timeout 300 python tools/solve_table.py 1 2 3 4 > gpurun_out/r2_solve_table4.jsonl 2>&1
timeout 300 python tools/size_sweep.py > gpurun_out/r2_size_sweep2.txt 2>&1
timeout 600 python tools/split_model.py > gpurun_out/r2_split_model.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tall5.log 2>&1
