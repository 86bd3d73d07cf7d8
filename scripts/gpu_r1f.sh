mkdir -p gpurun_out
timeout 300 python scripts/probe_tail.py > gpurun_out/tail_coop.log 2>&1
DROTB_TAIL=legacy timeout 300 python scripts/probe_tail.py > gpurun_out/tail_legacy.log 2>&1
echo "== coop"; cat gpurun_out/tail_coop.log; echo "== legacy"; cat gpurun_out/tail_legacy.log
for f in tests/test_tail_gpu.py tests/test_persistent_gpu.py tests/test_solve_gpu.py tests/test_shard_gpu.py tests/test_sweep_gpu.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  echo "$b: $(tail -2 gpurun_out/t_$b.log | head -1)"
done
DROTB_NO_GRAPHS=1 timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches_warm_coop.csv python scripts/ncu_probe.py 10000 f32 20 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -n 3 gpurun_out/bench.err
