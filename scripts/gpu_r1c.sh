mkdir -p gpurun_out
timeout 300 python scripts/probe_tail.py > gpurun_out/tail_p.log 2>&1
DROTB_PERSIST=0 timeout 300 python scripts/probe_tail.py > gpurun_out/tail_np.log 2>&1
for f in tests/test_persistent_gpu.py tests/test_pass_gpu.py tests/test_solve_gpu.py tests/test_shard_gpu.py tests/test_probgen_gpu.py tests/test_report_gpu.py tests/test_sweep_gpu.py tests/test_fullsize_gpu.py tests/test_dropin_gpu.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -m gpu -v -rf --timeout 300 --timeout-method=thread --durations=10 > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  echo "$b: $(grep -E '^(=+ .*(passed|failed|error).*=+)$' gpurun_out/t_$b.log | tail -1) $(tail -1 gpurun_out/t_$b.log)"
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 600 bash scripts/ncu_run.sh r1c 10000 f32
cat gpurun_out/tail_p.log gpurun_out/tail_np.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
