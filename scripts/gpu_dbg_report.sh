mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_report_gpu.py -m gpu -q -x -rf > gpurun_out/dbg1.log 2>&1; echo "rc $?" >> gpurun_out/dbg1.log; tail -5 gpurun_out/dbg1.log
timeout 600 python -m pytest tests/test_probgen_gpu.py tests/test_report_gpu.py -m gpu -q -x -rf > gpurun_out/dbg2.log 2>&1; echo "rc $?" >> gpurun_out/dbg2.log; tail -5 gpurun_out/dbg2.log
timeout 600 python -m pytest tests/test_persistent_gpu.py tests/test_probgen_gpu.py tests/test_report_gpu.py -m gpu -q -x -rf > gpurun_out/dbg3.log 2>&1; echo "rc $?" >> gpurun_out/dbg3.log; tail -5 gpurun_out/dbg3.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_report_gpu.py -m gpu -q -x -k "shape0 or shape1" > gpurun_out/dbg4.log 2>&1; echo "rc $?" >> gpurun_out/dbg4.log; tail -30 gpurun_out/dbg4.log
