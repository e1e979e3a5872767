#!/bin/bash
# 2/4-GPU: multi-rank tests, then C5 weak-scaling bench at K = 2 and K = 3 (far particles across ranks fused).
TAG=${1:-r2k}; N=${2:-2}
bash scripts/r2_multi.sh $TAG $N 1 0
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
P=29700
for K in 2 3; do
  P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus $N --steps 9 --warmup 3 --no-e2e --rebin-interval $K > gpurun_out/${TAG}_bench_K$K.log 2>&1
  L=$(grep '^{' gpurun_out/${TAG}_bench_K$K.log | tail -1)
  if [ -n "$L" ]; then echo "$L" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('bench K=$K %.4g pu/s  ms/step %.2f  frac %.3f  general %d  fused %d far %d' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['general_rebins'], j['fused_rebins'], j['far_last_rebin']))"; else echo "bench K=$K failed"; grep -m3 -i "error" gpurun_out/${TAG}_bench_K$K.log; fi
done
