#!/bin/bash
# Multi-GPU evidence on one box with N GPUs: multi-rank parity tests, the C5 weak-scaling
# bench line, and the clustered-load A/B of the decompositions.
# usage: bash scripts/r2_multi.sh <tag> <N> [tests=1] [benches=1]
TAG=${1:-r2m}; N=${2:-2}; TESTS=${3:-1}; BENCH=${4:-1}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
if [ "$TESTS" = 1 ]; then
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -o "MR_REPORT.*" gpurun_out/${TAG}_pytest.log | cut -c1-400
fi
[ "$BENCH" = 1 ] || exit 0
P=29600
run() {
  P=$((P+1))
  timeout 900 $TR --master-port $P bench.py --gpus $N --steps 8 --warmup 3 --no-e2e "$@" > gpurun_out/${TAG}_bench_${P}.log 2>&1
  rc=$?
  L=$(grep '^{' gpurun_out/${TAG}_bench_${P}.log | tail -1)
  if [ -n "$L" ]; then echo "$L" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('bench [$*] %.4g pu/s  ms/step %.2f  frac %.3f  general %d  fused %d' % (j['value'], j['ms_per_step'], j['roofline']['frac'], j['general_rebins'], j['fused_rebins']))"; else echo "bench [$*] rc=$rc"; grep -m2 "Error" gpurun_out/${TAG}_bench_${P}.log; fi
}
run
run --decomp sharded
for part in "--partition equal" "--partition weighted" "--decomp sharded" "--decomp sharded --partition hilbert"; do
  run --particles 4e8 --cluster 0.15 $part
done
