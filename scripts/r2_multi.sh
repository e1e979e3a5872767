#!/bin/bash
# Multi-GPU evidence on one box with N GPUs: multi-rank parity tests, the C5 weak-scaling
# bench line, and the clustered-load A/B of the decompositions.
# usage: bash scripts/r2_multi.sh <tag> <N>
TAG=${1:-r2m}; N=${2:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
P=29600
for args in "" "--decomp sharded" "--cluster 0.15 --partition equal" "--cluster 0.15 --partition weighted" "--cluster 0.15 --decomp sharded"; do
  P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus $N --steps 8 --warmup 3 --no-e2e $args > gpurun_out/${TAG}_bench_${P}.log 2>&1
  echo "bench [$args] rc=$?"; grep '^{' gpurun_out/${TAG}_bench_${P}.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('  value %.4g pu/s  ms/step %.2f  frac %.3f  general %d  fused %d' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['general_rebins'], j['fused_rebins']))"
done
