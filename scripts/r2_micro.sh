#!/bin/bash
# Droplet step (f3) evidence: GPU parity, timing of both arithmetic modes, one ncu
# --set full capture of each kernel flavour.  usage: bash scripts/r2_micro.sh <tag>
TAG=${1:-r2mi}
timeout 900 python -m pytest tests/test_gpu_micro.py -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
for ar in fp64 fp32; do for ns in 1 4; do
  timeout 600 python scripts/micro_timing.py --arith $ar --nsteps $ns > gpurun_out/${TAG}_time_${ar}_${ns}.log 2>&1
  echo "time $ar nsteps=$ns rc=$? $(grep '^{' gpurun_out/${TAG}_time_${ar}_${ns}.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print("%.3g upd/s %.2f ms/call %.0f GB/s" % (j["value"], j["ms_per_call"], j["achieved_GBs"]))')"
done; done
for ar in fp64 fp32; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_micro -c 1 -o gpurun_out/${TAG}_ncu_${ar} \
    python scripts/micro_timing.py --arith $ar --n 50000000 --calls 1 --warmup 0 > gpurun_out/${TAG}_ncu_${ar}.log 2>&1
  echo "ncu $ar rc=$?"
done
