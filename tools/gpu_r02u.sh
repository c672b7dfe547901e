#!/bin/bash
# ncu --set full of the persistent Ozaki GEMM (one CTA per tile and cluster-pair variants)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 1; do
  RBA_OZ_2CTA=$v timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_oz_gemm" \
    --launch-skip 30 --launch-count 3 -o gpurun_out/r02u_oz$v python tools/oz_check.py > gpurun_out/r02u_oz$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r02u_oz$v.log
done
