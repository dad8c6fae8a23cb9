set -x
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-solve > gpurun_out/r2p_bench_default_$i.json 2> /dev/null
cp paper_1301_5914_b200/libhobi.so /tmp/libhobi_default.so
cp tools/_libhobi_O1.so paper_1301_5914_b200/libhobi.so
timeout 600 python bench.py --no-cpu-baseline --no-solve > gpurun_out/r2p_bench_O1_$i.json 2> gpurun_out/r2p_bench_O1.err
cp /tmp/libhobi_default.so paper_1301_5914_b200/libhobi.so
done
