#!/bin/bash
# ncu per-launch metrics of the step and rebin kernels at C3 (1e8 on 256^3, K = 4).
TAG=${1:-r2c3m}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --metrics $M --clock-control none --csv -k regex:"^k_" -s 40 -c 60 --log-file gpurun_out/${TAG}_C3_metrics.csv \
  python bench.py --workload C3 --steps 8 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > gpurun_out/${TAG}_C3.log 2>&1
echo "ncu rc=$?"
