mkdir -p gpurun_out
timeout 300 python scripts/probe_tail.py > gpurun_out/tail_p3.log 2>&1
DROTB_PSK_SCHED=f timeout 300 python scripts/probe_tail.py > gpurun_out/tail_p3f.log 2>&1
cat gpurun_out/tail_p3.log gpurun_out/tail_p3f.log
for f in tests/test_persistent_gpu.py tests/test_solve_gpu.py tests/test_pass_gpu.py tests/test_shard_gpu.py tests/test_probgen_gpu.py tests/test_report_gpu.py tests/test_sweep_gpu.py tests/test_fullsize_gpu.py tests/test_dropin_gpu.py; do
  b=$(basename $f .py)
  timeout 600 python -m pytest $f -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/t_$b.log 2>&1; echo "rc $?" >> gpurun_out/t_$b.log
  echo "$b: $(tail -2 gpurun_out/t_$b.log | head -1)"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 -o gpurun_out/solve_r1e python scripts/ncu_probe.py 10000 f32 6 2 > gpurun_out/p_r1e.log 2>&1
