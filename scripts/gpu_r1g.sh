mkdir -p gpurun_out
timeout 300 python scripts/probe_tail.py > gpurun_out/tail_coop2.log 2>&1
cat gpurun_out/tail_coop2.log
for f in tests/test_tail_gpu.py tests/test_solve_gpu.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  echo "$b: $(tail -2 gpurun_out/t_$b.log | head -1)"
done
DROTB_NO_GRAPHS=1 timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches_warm_coop2.csv python scripts/ncu_probe.py 10000 f32 20 > /dev/null 2>&1
DROTB_NO_GRAPHS=1 timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:tail_kernel -s 6 -c 2 -o gpurun_out/tail_r1g python scripts/ncu_probe.py 10000 f32 12 > gpurun_out/p_r1g.log 2>&1
