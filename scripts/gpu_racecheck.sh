for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_tail_gpu.py -m gpu -q -x -k "cluster_tail_equals_grid_tail and shape0" --timeout 900 > gpurun_out/${tool}_tail.log 2>&1; echo "rc $?" >> gpurun_out/${tool}_tail.log
done
