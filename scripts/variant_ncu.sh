#!/bin/bash
# ncu DRAM / L2 / stall metrics of k_fs for each build in build/variants (one GPU).
NP=${1:-4e8}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
cp paper_2603_26691_b200/lib/libscaletrack.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  cp $v paper_2603_26691_b200/lib/libscaletrack.so
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_fs" -s 2 -c 1 --log-file gpurun_out/vn_$(basename $v .so).csv \
    python bench.py --particles $NP --steps 2 --warmup 3 --no-cpu-baseline --no-micro --no-e2e > /dev/null 2>&1
  echo "$v rc=$?"; grep -E "dram__bytes|gpu__time|issue_active|stalled" gpurun_out/vn_$(basename $v .so).csv | awk -F'","' '{print $(NF-2), $NF}'
done
cp /tmp/lib_orig.so paper_2603_26691_b200/lib/libscaletrack.so
