mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_tail_gpu.py tests/test_iter_gpu.py -m gpu -q -x -k "graphs_equal or mid_run or l2_policies or vcta or fixed_iterations" > gpurun_out/mc2.log 2>&1; echo "rc $?" >> gpurun_out/mc2.log
grep -E "ERROR SUMMARY|passed|failed|^rc|Invalid" gpurun_out/mc2.log | head -20
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_solve_gpu.py -m gpu -q -x -k "edge or drot_step or validation" > gpurun_out/mc3.log 2>&1; echo "rc $?" >> gpurun_out/mc3.log
grep -E "ERROR SUMMARY|passed|failed|^rc|Invalid" gpurun_out/mc3.log | head -20
