#!/bin/bash
# One-GPU round-2 evidence: pytest -m gpu, smoke, bench lines (C5 default, K=3, C3, C4),
# the coupling-buffer timeline.  usage: bash scripts/r2_single.sh <tag>
TAG=${1:-r2s}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/${TAG}_smoke.log)"
b() {
  name=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1
  rc=$?; L=$(grep '^{' gpurun_out/${TAG}_bench_${name}.log | tail -1)
  if [ -n "$L" ]; then echo "$L" | python -c "import json,sys; j=json.loads(sys.stdin.read()); e=j.get('e2e') or {}; c=j.get('cpu_baseline') or {}; print('bench $name: %.4g pu/s  ms/step %.2f  frac %.3f  e2e %s  far %s  general %d  cpu %s' % (j['value'], j['ms_per_step'], j['roofline']['frac'], e.get('value'), j.get('far_last_rebin'), j['general_rebins'], c.get('value')))"; else echo "bench $name rc=$rc"; tail -3 gpurun_out/${TAG}_bench_${name}.log; fi
}
b C5 --steps 20 --warmup 3
b C5K3 --steps 12 --warmup 3 --rebin-interval 3 --no-cpu-baseline --no-micro
b C3 --workload C3 --steps 20 --warmup 3 --no-micro
b C4 --workload C4 --steps 10 --warmup 3 --no-micro --no-cpu-baseline
timeout 900 python scripts/coupling_timeline.py --workload C3 --steps 12 --out gpurun_out/${TAG}_timeline_c3.json > gpurun_out/${TAG}_timeline_c3.log 2>&1
echo "timeline rc=$?"; tail -2 gpurun_out/${TAG}_timeline_c3.log
timeout 900 python scripts/coupling_timeline.py --workload C5 --steps 8 --out gpurun_out/${TAG}_timeline_c5.json > gpurun_out/${TAG}_timeline_c5.log 2>&1
echo "timeline c5 rc=$?"; tail -1 gpurun_out/${TAG}_timeline_c5.log
