mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests.log
tail -25 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log; cat gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -n 3 gpurun_out/bench.err
