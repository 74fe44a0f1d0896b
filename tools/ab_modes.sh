#!/bin/bash
mkdir -p gpurun_out
for m in 0 1; do
  TCB_QUERY_MODE=$m timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/ab_mode$m.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_mode$m.json'));print('mode',$m,d['ms_per_step'],d['stage_ms'])"
done
TCB_QUERY_MODE=0 timeout 900 tools/profile.sh r01b k_fd_main > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r01b_k_fd_main_raw.csv')))
hdr=rows[0]
for name in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__thread_inst_executed_per_inst_executed.ratio','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread']:
    if name in hdr:
        i=hdr.index(name); print(name, rows[1][i], rows[2][i])
PY
