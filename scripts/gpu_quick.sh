#!/bin/bash
# Quick iteration loop on a GPU box: timeline probe, a test subset, a short
# bench (no extras).  usage: scripts/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-"tail or golden_fast or api or dropin or c4_grid_fast or golden_c2"}
mkdir -p gpurun_out
timeout 300 python scripts/probe_timeline.py 10000 f32 > gpurun_out/timeline_${TAG}.log 2>&1
timeout 300 python scripts/probe_timeline.py 1000 f64 >> gpurun_out/timeline_${TAG}.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-c5 --no-sinkhorn --no-f64 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/tests_${TAG}.log 2>&1
cat gpurun_out/timeline_${TAG}.log; tail -3 gpurun_out/tests_${TAG}.log; tail -2 gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['time_to_tol_c2']['ms_per_iteration'], d['time_to_tol_c2']['iterations'])"
