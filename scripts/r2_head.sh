#!/bin/bash
# Re-entry check at HEAD: GPU tests, smoke, default bench line, droplet-step timing.
TAG=${1:-r2u}
bash scripts/r2_single2.sh $TAG "test"
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_C5.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/${TAG}_bench_C5.log | head -c 600; echo
for ar in fp64 fp32; do
  timeout 600 python scripts/micro_timing.py --arith $ar --nsteps 1 --calls 8 > gpurun_out/${TAG}_t_${ar}.log 2>&1
  echo "micro $ar rc=$? $(grep '^{' gpurun_out/${TAG}_t_${ar}.log | head -c 300)"
done
