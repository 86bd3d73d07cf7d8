mkdir -p gpurun_out
for f in test_report_gpu test_probgen_gpu test_sinkhorn_gpu test_solve_gpu test_pass_gpu test_sweep_gpu; do
  timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/$f.py -m gpu -q -x --timeout 600 > gpurun_out/mc_$f.log 2>&1; echo "rc $?" >> gpurun_out/mc_$f.log
  echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|^rc" gpurun_out/mc_$f.log | tail -4
done
