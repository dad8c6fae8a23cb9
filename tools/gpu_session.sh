set -x
timeout 900 python -m pytest tests/test_gpu_singular.py -q -x > gpurun_out/r2m_singular.txt 2>&1
for c in 1 4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:singular --csv --log-file gpurun_out/r2m_launch_c$c.csv python tools/launch_breakdown.py $c > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r2m_launch_c$c.csv > gpurun_out/r2m_launch_summary_c$c.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:singular_fast -s 2 -c 1 -o gpurun_out/r2m_singular_c4 python tools/launch_breakdown.py 4 > gpurun_out/r2m_ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2m_gputest.txt 2>&1; echo "gputest rc=$?" >> gpurun_out/r2m_gputest.txt
timeout 600 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
