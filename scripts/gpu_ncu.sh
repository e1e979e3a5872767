#!/bin/bash
# ncu captures of the step kernel and the rebin prep (1 GPU).
# usage: bash scripts/gpu_ncu.sh <tag> [particles]
TAG=${1:-r}
NP=${2:-2e7}
CMD="python bench.py --particles $NP --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${EXTRA}"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
echo "launch list rc=$?"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_pstep|k_step|k_rebin_prep}" -s ${SKIP:-2} -c ${CNT:-3} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
