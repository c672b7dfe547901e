#!/bin/bash
# ncu --set full of the LONGEST k_oz_gemm launch of one C4 factorisation batch (a top-level
# Schur update): pass 1 lists the launch durations, pass 2 captures that launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"^k_oz_gemm$" -c 260 --csv \
  --log-file gpurun_out/ozbig_list.csv python tools/oz_check.py > gpurun_out/ozbig_list.log 2>&1
IDX=$(python - <<'PY'
import csv
rows=[l for l in open('gpurun_out/ozbig_list.csv') if not l.startswith('==')]
d=[float(r['Metric Value'].replace(',','')) for r in csv.DictReader(rows)]
i=max(range(len(d)), key=lambda k:d[k])
print(i)
PY
)
echo "longest k_oz_gemm launch: index $IDX"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"^k_oz_gemm$" \
  --launch-skip $IDX --launch-count 1 -o gpurun_out/ozbig_full -f python tools/oz_check.py > gpurun_out/ozbig_full.log 2>&1
echo "full rc=$?"
