#!/bin/bash
# 4-GPU box: all GPU tests (single- and multi-rank), then C5 weak-scaling lines at N = 4 and 2.
TAG=${1:-r2m4}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
bash scripts/r2_mk.sh ${TAG}n4 4 "${2:-3 4}"
