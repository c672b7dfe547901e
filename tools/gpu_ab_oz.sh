#!/bin/bash
# A/B of Ozaki GEMM variants on the C4 factorisation: env assignments per run, e.g.
#   bash tools/gpu_ab_oz.sh "RBA_OZ_TS=0" "RBA_OZ_TS=1" "RBA_OZ_TS=1 RBA_OZ_STAGES=5"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  env $cfg timeout 600 python tools/oz_check.py > gpurun_out/ab_oz_$i.log 2>&1
  echo "== $cfg"; grep -h "oz_prof\|factor 16\|classes" gpurun_out/ab_oz_$i.log | cut -c1-420
  i=$((i+1))
done
