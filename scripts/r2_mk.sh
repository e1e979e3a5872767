#!/bin/bash
# Multi-GPU C5 bench lines at several rebin intervals with the timeline of the calls.
# usage: bash scripts/r2_mk.sh <tag> <N> "<K list>" [tests]
TAG=${1:-r2mk}; N=${2:-2}; KS=${3:-"2 3"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
if [ "$4" == "tests" ]; then
  timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
fi
P=29700
for K in $KS; do
  P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus $N --steps 18 --warmup 3 --no-e2e --rebin-interval $K > gpurun_out/${TAG}_K$K.log 2>&1
  grep '^{' gpurun_out/${TAG}_K$K.log | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); s=j['step_kernel_ms_series']
print('N=$N K=$K %.4g pu/s %.3f ms/step frac %.3f far %s gen %s reb %.2f timeline %s series %s..%s' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['far_last_rebin'], j['general_rebins'], j['rebin_prep_ms'], json.dumps(j.get('timeline')), s[:$K], s[-$K:]))" || tail -5 gpurun_out/${TAG}_K$K.log
done
