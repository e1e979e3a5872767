#!/bin/bash
# N-GPU round-2 evidence: multi-rank tests, C5 at K = 2 and 3, the clustered A/B.
TAG=${1:-r2q}; N=${2:-4}
bash scripts/r2_multi.sh $TAG $N 1 0
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
P=29800
run() {
  name=$1; shift; P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus $N --steps 9 --warmup 3 --no-e2e "$@" > gpurun_out/${TAG}_bench_$name.log 2>&1
  L=$(grep '^{' gpurun_out/${TAG}_bench_$name.log | tail -1)
  if [ -n "$L" ]; then echo "$L" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('bench $name %.4g pu/s  ms/step %.2f  frac %.3f  general %d  fused %d far %d' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['general_rebins'], j['fused_rebins'], j['far_last_rebin']))"; else echo "bench $name failed"; grep -m3 -i "error" gpurun_out/${TAG}_bench_$name.log; fi
}
run K2 --rebin-interval 2
run K3 --rebin-interval 3
run sharded --decomp sharded --rebin-interval 2
for part in "equal" "weighted"; do run cl_$part --particles 2e8 --cluster 0.15 --partition $part --rebin-interval 2; done
run cl_sharded --particles 2e8 --cluster 0.15 --decomp sharded --rebin-interval 2
run cl_hilbert --particles 2e8 --cluster 0.15 --decomp sharded --partition hilbert --rebin-interval 2
