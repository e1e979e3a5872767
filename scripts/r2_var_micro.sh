#!/bin/bash
# k_fs warp-count variants (bench A/B) + droplet-step timing diagnostics with clocks.
TAG=${1:-r2vm}
timeout 600 python -m pytest tests/test_gpu_micro.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_micro.log 2>&1; echo "pytest micro rc=$? $(tail -1 gpurun_out/${TAG}_pytest_micro.log)"
bash scripts/variants.sh --steps 8 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_variants.log 2>&1
cat gpurun_out/${TAG}_variants.log
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 250 > gpurun_out/${TAG}_smi.csv &
SMI=$!
for rep in 1 2; do for ar in fp64 fp32; do for ns in 1 4; do
  timeout 600 python scripts/micro_timing.py --arith $ar --nsteps $ns --calls 8 > gpurun_out/${TAG}_t_${ar}_${ns}_${rep}.log 2>&1
  echo "$(date +%T) time $ar nsteps=$ns rep=$rep rc=$? $(grep '^{' gpurun_out/${TAG}_t_${ar}_${ns}_${rep}.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print("%.3g upd/s %.2f ms/call per-call %s" % (j["value"], j["ms_per_call"], [round(v,1) for v in j["per_call_ms"]]))')"
done; done; done
kill $SMI
