#!/bin/bash
# 2-GPU box at HEAD: multi-rank GPU tests and the C5 K = 4 weak-scaling line at N = 2.
TAG=${1:-r2m2f}
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest multirank rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
bash scripts/r2_mk.sh ${TAG}n2 2 "4"
