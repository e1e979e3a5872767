#!/bin/bash
# Round-end evidence on one GPU: default bench line, its ncu launch list, and the DRAM
# traffic of one step-kernel launch at the headline size (no --set full replay at 1e9:
# two DRAM counters fit one pass).
# usage: bash scripts/gpu_final.sh <tag>
TAG=${1:-r1}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch list rc=$?"
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:"k_pstep|k_count" -s 6 -c 6 --log-file gpurun_out/traffic_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_traffic_$TAG.log 2>&1; echo "ncu traffic rc=$?"
