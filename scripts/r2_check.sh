#!/bin/bash
# GPU tests (optionally a -k filter) then a rebin-interval sweep with the in-tree build.
# usage: bash scripts/r2_check.sh <tag> "<pytest -k expr or all>" "<sweep cases>"
TAG=${1:-r2c}; KEXPR=${2:-all}; CASES=${3:-"C5:3 C5:4 C3:4"}
if [ "$KEXPR" == "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$KEXPR" > gpurun_out/${TAG}_pytest.log 2>&1
fi
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED|^E " gpurun_out/${TAG}_pytest.log | head -12
[ -n "$CASES" ] && bash scripts/r2_ksweep.sh $TAG "$CASES"
