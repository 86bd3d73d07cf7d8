#!/bin/bash
# ${TAG:-r2b}: verification of the split host driver + the C2 golden (order=reference to 1e-4)
TAG=${1:-r2b}
bash scripts/gpu_round.sh $TAG
timeout 1500 python tests/golden/make_c2_golden.py gpurun_out/golden > gpurun_out/golden_c2.log 2>&1
echo "golden rc $?" >> gpurun_out/golden_c2.log
tail -3 gpurun_out/golden_c2.log
