#!/bin/bash
# One-GPU round-2 evidence, second pass: tests, smoke, bench lines, timelines, ncu
# metrics and compute-sanitizer.  usage: bash scripts/r2_single2.sh <tag> [parts]
TAG=${1:-r2t}; PARTS=${2:-"test bench timeline metrics sanitize"}
b() {
  name=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1
  rc=$?; L=$(grep '^{' gpurun_out/${TAG}_bench_${name}.log | tail -1)
  if [ -n "$L" ]; then echo "$L" | python -c "import json,sys; j=json.loads(sys.stdin.read()); e=j.get('e2e') or {}; c=j.get('cpu_baseline') or {}; print('bench $name: %.4g pu/s  ms/step %.2f  frac %.3f  e2e %s  far %s  general %d  cpu %s' % (j['value'], j['ms_per_step'], j['roofline']['frac'], e.get('value'), j.get('far_last_rebin'), j['general_rebins'], c.get('value')))"; else echo "bench $name rc=$rc"; tail -3 gpurun_out/${TAG}_bench_${name}.log; fi
}
for part in $PARTS; do case $part in
test)
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$? $(tail -1 gpurun_out/${TAG}_smoke.log)" ;;
bench)
  b C5 --steps 20 --warmup 3
  b C5K2 --steps 12 --warmup 3 --rebin-interval 2 --no-cpu-baseline --no-micro
  b C5K3 --steps 12 --warmup 3 --rebin-interval 3 --no-cpu-baseline --no-micro ;;
timeline)
  for W in C3 C5; do
    timeout 900 python scripts/coupling_timeline.py --workload $W --steps 12 --out gpurun_out/${TAG}_timeline_$W.json > gpurun_out/${TAG}_timeline_$W.log 2>&1
    echo "timeline $W rc=$?"; tail -1 gpurun_out/${TAG}_timeline_$W.log
  done ;;
metrics)
  bash scripts/r2_metrics.sh ${TAG}m C5
  bash scripts/r2_metrics.sh ${TAG}m C3 ;;
sanitize)
  for tool in memcheck racecheck synccheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/${TAG}_sanitize_$tool.log 2>&1
    echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_CASE_OK' gpurun_out/${TAG}_sanitize_$tool.log | tr '\n' ' ')"
  done ;;
esac; done
