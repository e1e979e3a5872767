#!/bin/bash
# ncu --set full of the two k_pstep flavours (fused scatter + in-place counting).
# usage: bash scripts/r2_prof.sh <tag> [particles]
TAG=${1:-r2}
NP=${2:-4e8}
CMD="python bench.py --particles $NP --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-micro"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"; tail -c 1500 gpurun_out/${TAG}_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_pstep}" -s ${SKIP:-2} -c ${CNT:-2} \
  -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
