#!/bin/bash
# Round-2 final single-GPU evidence at HEAD: tests, smoke, default bench line (K = 4),
# C4 / C3 lines, coupling timelines, ncu metrics at C5 1e9 (traffic, L2 hit, reductions),
# ncu --set full of the two step kernels at 4e8, a launch list.  usage: bash scripts/r2_final.sh <tag> [parts]
TAG=${1:-r2v2}; PARTS=${2:-"test bench timeline metrics full launches"}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for part in $PARTS; do case $part in
test)
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"; grep -E "^FAILED" gpurun_out/${TAG}_pytest.log | head
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$? $(tail -1 gpurun_out/${TAG}_smoke.log)" ;;
bench)
  timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_C5.log 2>&1; echo "bench C5 rc=$?"
  grep '^{' gpurun_out/${TAG}_bench_C5.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['ms_per_step'], j['roofline']['frac'], j['roofline']['traffic'], json.dumps(j['e2e'])[:600], j['clocks'], (j.get('micro_f3') or {}).get('fp32'))"
  for W in C4 C3; do
    timeout 1200 python bench.py --workload $W --steps 20 --warmup 3 --no-micro > gpurun_out/${TAG}_bench_$W.log 2>&1; echo "bench $W rc=$?"
    grep '^{' gpurun_out/${TAG}_bench_$W.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['ms_per_step'], j['roofline']['frac'], (j['e2e'] or {}).get('value'), j['rebin_prep_ms'])"
  done ;;
timeline)
  for W in C3 C5; do
    timeout 900 python scripts/coupling_timeline.py --workload $W --steps 12 --out gpurun_out/${TAG}_timeline_$W.json > gpurun_out/${TAG}_timeline_$W.log 2>&1
    echo "timeline $W rc=$?"; tail -1 gpurun_out/${TAG}_timeline_$W.log
  done ;;
metrics)
  timeout 1500 ncu --metrics $M --clock-control none --csv -k regex:"k_fs|k_ip|k_rebin_prep|k_dbase|k_far_order|k_field_ingest|k_source_readout|k_items|k_scan" \
    -s 60 -c 24 --log-file gpurun_out/${TAG}_C5_metrics.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_C5_metrics.log 2>&1
  echo "ncu metrics rc=$?"
  python scripts/traffic_json.py gpurun_out/${TAG}_C5_metrics.csv 1e9 4 "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_red.sum --clock-control none, C5 1e9 particles, K = 4 (profiles/r2/${TAG}_C5_metrics.csv); per launch" ;;
full)
  CMD="python bench.py --particles 4e8 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-micro"
  for K in k_fs k_ip; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
    echo "ncu full $K rc=$?"
  done ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/${TAG}_launches_C5.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_launches.log 2>&1
  echo "launches rc=$?" ;;
esac; done
