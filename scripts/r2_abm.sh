#!/bin/bash
# Multi-GPU A/B of library variants (build/variants/*.so): C5 weak scaling bench at N GPUs.
# usage: bash scripts/r2_abm.sh <tag> <N> "<bench args>"
TAG=${1:-r2abm}; N=${2:-2}; ARGS=${3:-"--steps 12 --warmup 3 --no-e2e"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
cp paper_2603_26691_b200/lib/libscaletrack.so /tmp/lib_orig.so
P=29800
for v in build/variants/*.so; do
  P=$((P+1))
  cp $v paper_2603_26691_b200/lib/libscaletrack.so
  timeout 900 $TR --master-port $P bench.py --gpus $N $ARGS > gpurun_out/${TAG}_$(basename $v .so).log 2>&1
  grep '^{' gpurun_out/${TAG}_$(basename $v .so).log | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); s=j['step_kernel_ms_series']
print('$v N=$N %.4g pu/s %.3f ms/step reb %.2f series %s..%s' % (j['value'], j['ms_per_step'], j['rebin_prep_ms'], s[:4], s[-4:]))" || tail -3 gpurun_out/${TAG}_$(basename $v .so).log
done
cp /tmp/lib_orig.so paper_2603_26691_b200/lib/libscaletrack.so
