set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2n_gputest.txt 2>&1; echo "gputest rc=$?" >> gpurun_out/r2n_gputest.txt
timeout 600 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
HOBI_FORCE_NCCL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_torchrun_n1.json 2> gpurun_out/r2n_torchrun_n1.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.txt 2>&1
