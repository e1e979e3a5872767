#!/bin/bash
# Source-level ncu of the two step kernels (k_fs fused, k_ip in place) at a reduced
# particle count, plus a default bench line (e2e diagnostics).  usage: bash scripts/r2_src_prof.sh <tag> [particles]
TAG=${1:-r2v}; NP=${2:-4e8}
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-micro > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?"; grep '^{' gpurun_out/${TAG}_bench.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step'], j['roofline']['frac'], json.dumps(j['e2e']), json.dumps(j['clocks']))"
CMD="python bench.py --particles $NP --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-micro"
for K in k_fs k_ip; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 \
    -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
  echo "ncu $K rc=$?"; tail -2 gpurun_out/${TAG}_ncu_$K.log
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${K}_sass.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_${K}_cuda.csv 2>/dev/null
  ls -la gpurun_out/${TAG}_${K}*
done
