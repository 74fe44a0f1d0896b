#!/bin/bash
# A/B of the main-pass traversal variants: bench stage times + key ncu counters.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
MET=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__warps_eligible.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio
for t in down up; do
  for m in 0 1; do
    TCB_MAIN_TRAVERSAL=$t TCB_QUERY_MODE=$m timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/abt_${t}_$m.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/abt_${t}_$m.json'));print('$t mode $m', d['ms_per_step'], d['stage_ms']['main'])"
  done
  TCB_MAIN_TRAVERSAL=$t $NCU --metrics $MET --clock-control none -k regex:k_fd_main -c 1 --csv python bench.py --no-cpu-baseline --steps 1 2>/dev/null | grep -E '"(gpu__time|smsp__inst|smsp__thread|dram__bytes|lts__t|l1tex__t|smsp__warps|sm__warps|smsp__average)' | awk -F'","' '{print "'$t'", $(NF-2), $NF}'
done
