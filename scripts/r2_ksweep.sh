#!/bin/bash
# Rebin-interval sweep on one GPU.  usage: bash scripts/r2_ksweep.sh <tag> "<workload:K ...>"
TAG=${1:-r2k}; CASES=${2:-"C5:2 C5:3 C5:4 C3:2 C3:3 C3:4"}
for c in $CASES; do
  W=${c%%:*}; K=${c##*:}
  timeout 900 python bench.py --workload $W --rebin-interval $K --steps 24 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_${W}_K$K.log 2>&1
  grep '^{' gpurun_out/${TAG}_${W}_K$K.log | python -c "
import json,sys; j=json.loads(sys.stdin.read()); s=j['step_kernel_ms_series']
print('$W K=$K %.4g pu/s %.3f ms/step frac %.3f far %s general %s rebin %.2f ms series %s..%s' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['far_last_rebin'], j['general_rebins'], j['rebin_prep_ms'], s[:$K], s[-$K:]))" || tail -3 gpurun_out/${TAG}_${W}_K$K.log
done
