#!/bin/bash
# compute-sanitizer over the GPU tests (memcheck), and racecheck / synccheck
# on the tail tests (cluster tail: DSMEM reductions, cluster barriers)
mkdir -p gpurun_out
for f in test_tail_gpu test_report_gpu test_probgen_gpu test_sinkhorn_gpu test_solve_gpu test_pass_gpu test_sweep_gpu; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/$f.py -m gpu -q -x --timeout 900 > gpurun_out/mc_$f.log 2>&1; echo "rc $?" >> gpurun_out/mc_$f.log
  echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|^rc" gpurun_out/mc_$f.log | tail -4
done
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_tail_gpu.py -m gpu -q -x -k "cluster_tail_equals_grid_tail and shape0" --timeout 900 > gpurun_out/${tool}_tail.log 2>&1; echo "rc $?" >> gpurun_out/${tool}_tail.log
  echo "== $tool tail"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|^rc" gpurun_out/${tool}_tail.log | tail -4
done
