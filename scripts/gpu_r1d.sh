mkdir -p gpurun_out
timeout 120 ./scripts/barrier_bench > gpurun_out/barrier.log 2>&1
timeout 300 python scripts/probe_tail.py > gpurun_out/tail_p2.log 2>&1
DROTB_PERSIST=0 timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_warm_np.csv python scripts/ncu_probe.py 10000 f32 20 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 -o gpurun_out/solve_r1d python scripts/ncu_probe.py 10000 f32 6 2 > gpurun_out/p_r1d.log 2>&1
for f in tests/test_persistent_gpu.py tests/test_solve_gpu.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  echo "$b: $(tail -2 gpurun_out/t_$b.log | head -1)"
done
cat gpurun_out/barrier.log gpurun_out/tail_p2.log
