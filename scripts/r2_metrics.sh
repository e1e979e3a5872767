#!/bin/bash
# Round-2 evidence on one GPU: per-kernel DRAM traffic, L2 hit rate, global reduction /
# atomic sectors and duration of the step kernels at a workload's full size (no
# --set full replay at 1e9: these counters fit a few passes), plus the bench line.
# usage: bash scripts/r2_metrics.sh <tag> <workload> [extra bench args]
TAG=${1:-r2}; WL=${2:-C5}; shift 2; EXTRA="$@"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
timeout 900 python bench.py --workload $WL --steps 8 --warmup 3 --no-micro $EXTRA > gpurun_out/${TAG}_${WL}_bench.log 2>&1
echo "bench rc=$?"; grep '^{' gpurun_out/${TAG}_${WL}_bench.log | tail -1 | cut -c1-1500
timeout 1500 ncu --metrics $M --clock-control none --csv -k regex:"k_fs|k_ip|k_pstep|k_count|k_rebin_prep|k_dbase|k_far_order|k_field_ingest|k_source_readout" \
  -s 30 -c 14 --log-file gpurun_out/${TAG}_${WL}_metrics.csv \
  python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu-baseline --no-micro --no-e2e $EXTRA > gpurun_out/${TAG}_${WL}_ncu.log 2>&1
echo "ncu metrics rc=$?"
