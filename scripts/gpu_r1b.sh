mkdir -p gpurun_out
timeout 300 python scripts/probe_tail.py > gpurun_out/tail.log 2>&1
DROTB_K1=r timeout 300 python scripts/probe_tail.py > gpurun_out/tail_r.log 2>&1
DROTB_NO_GRAPHS=1 timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_warm.csv python scripts/ncu_probe.py 10000 f32 20 > /dev/null 2>&1
for f in tests/test_dropin_gpu.py tests/test_probgen_gpu.py tests/test_pass_gpu.py tests/test_shard_gpu.py tests/test_solve_gpu.py tests/test_sweep_gpu.py tests/test_fullsize_gpu.py; do
  b=$(basename $f .py)
  timeout 900 python -m pytest $f -m gpu -v -rf --timeout 180 --durations=15 > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  tail -1 gpurun_out/t_$b.log
done
cat gpurun_out/tail.log gpurun_out/tail_r.log
