#!/bin/bash
# One verification pass on a GPU box: GPU tests, smoke, the bench at the
# driver's settings, ncu launch list + captures.  usage: scripts/gpu_round.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/gpu_tests_${TAG}.log 2>&1
echo "pytest rc $?" >> gpurun_out/gpu_tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc $?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc $?" >> gpurun_out/bench_${TAG}.err
tail -3 gpurun_out/gpu_tests_${TAG}.log; tail -2 gpurun_out/smoke_${TAG}.log; tail -3 gpurun_out/bench_${TAG}.err
