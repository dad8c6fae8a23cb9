for c in 1 2 4; do timeout 600 python tools/tune_sweep.py $c > gpurun_out/r2_tune2_c$c.txt 2>&1; done
